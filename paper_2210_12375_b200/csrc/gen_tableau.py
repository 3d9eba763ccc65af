"""Generate ``tableau_coeffs.h``: the embedded RK pairs as exact binary64.

The coefficients are the published ones (Dormand & Prince 1980; Tsitouras
2011, interpolant in its published factored form), written as hex-float
literals so the CUDA kernels, the C-ABI unit ops and the CPU oracle all see
the same bits as the reference's NumPy tables (reference
``pkg/src/batchode/tableau.py:102-149`` dopri5, ``:152-254`` tsit5, with the
tsit5 interpolant expanded by ``np.polymul`` exactly as ``tableau.py:86-99``
describes).  ``tests/test_oracle_golden.py`` checks every generated value
against the reference tableau dumped in ``tests/golden/tableaus.npz``.

The Heun-Euler pair is not in the reference; its data follows SURVEY.md
§8(b) (c=[0,1], a10=1, b=[1/2,1/2], b_err=[-1/2,1/2], interpolant
w0=theta-theta^2/2, w1=theta^2/2, non-FSAL).

    python paper_2210_12375_b200/csrc/gen_tableau.py
"""

import os

import numpy as np


def dopri5():
    a = np.zeros((7, 7))
    a[1, :1] = [1 / 5]
    a[2, :2] = [3 / 40, 9 / 40]
    a[3, :3] = [44 / 45, -56 / 15, 32 / 9]
    a[4, :4] = [19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729]
    a[5, :5] = [9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656]
    a[6, :6] = [35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84]
    b = np.append(a[6, :6], 0.0)
    b_err = np.array([71 / 57600, 0.0, -71 / 16695, 71 / 1920, -17253 / 339200,
                      22 / 525, -1 / 40])
    c = np.array([0.0, 1 / 5, 3 / 10, 4 / 5, 8 / 9, 1.0, 1.0])
    # Shampine's 4th-order continuous extension of DP5 (ascending theta^1..theta^4)
    interp = np.array([
        [1.0, -8048581381 / 2820520608, 8663915743 / 2820520608, -12715105075 / 11282082432],
        [0.0, 0.0, 0.0, 0.0],
        [0.0, 131558114200 / 32700410799, -68118460800 / 10900136933, 87487479700 / 32700410799],
        [0.0, -1754552775 / 470086768, 14199869525 / 1410260304, -10690763975 / 1880347072],
        [0.0, 127303824393 / 49829197408, -318862633887 / 49829197408, 701980252875 / 199316789632],
        [0.0, -282668133 / 205662961, 2019193451 / 616988883, -1453857185 / 822651844],
        [0.0, 40617522 / 29380423, -110615467 / 29380423, 69997945 / 29380423],
    ])
    return dict(S=7, a=a, b=b, b_err=b_err, c=c, interp=interp, order=5, error_order=4, fsal=1)


def tsit5():
    a = np.zeros((7, 7))
    a[1, :1] = [0.161]
    a[2, :2] = [-0.008480655492356989, 0.335480655492357]
    a[3, :3] = [2.8971530571054935, -6.359448489975075, 4.3622954328695815]
    a[4, :4] = [5.325864828439257, -11.748883564062828, 7.4955393428898365,
                -0.09249506636175525]
    a[5, :5] = [5.86145544294642, -12.92096931784711, 8.159367898576159,
                -0.071584973281401, -0.028269050394068383]
    a[6, :6] = [0.09646076681806523, 0.01, 0.4798896504144996, 1.379008574103742,
                -3.290069515436081, 2.324710524099774]
    b = np.append(a[6, :6], 0.0)
    b_err = np.array([-0.00178001105222577714, -0.0008164344596567469,
                      0.007880878010261995, -0.1447110071732629, 0.5823571654525552,
                      -0.45808210592918697, 0.015151515151515152])
    c = np.array([0.0, 0.161, 0.327, 0.9, 0.9800255409045097, 1.0, 1.0])
    th = np.array([1.0, 0.0])
    th2 = np.array([1.0, 0.0, 0.0])
    factored = [
        [np.array([-1.0530884977290216]), np.array([1.0, -1.3299890189751412]),
         np.array([1.0, -1.4364028541716351, 0.7139816917074209]), th],
        [np.array([0.1017]), np.array([1.0, -2.1966568338249754, 1.2949852507374631]), th2],
        [np.array([2.490627285651252793]), np.array([1.0, -2.38535645472061657, 1.57803468208092486]), th2],
        [np.array([-16.54810288924490272]), np.array([1.0, -1.21712927295533244]),
         np.array([1.0, -0.61620406037800089]), th2],
        [np.array([47.37952196281928122]), np.array([1.0, -1.203071208372362603]),
         np.array([1.0, -0.658047292653547382]), th2],
        [np.array([-34.87065786149660974]), np.array([1.0, -1.2]),
         np.array([1.0, -0.666666666666666667]), th2],
        [np.array([2.5]), np.array([1.0, -1.0]), np.array([1.0, -0.6]), th2],
    ]
    rows = []
    for factors in factored:
        poly = np.array([1.0])
        for fac in factors:
            poly = np.polymul(poly, fac)
        assert poly[-1] == 0.0
        rows.append(poly[:-1][::-1])
    return dict(S=7, a=a, b=b, b_err=b_err, c=c, interp=np.array(rows), order=5,
                error_order=4, fsal=1)


def heun():
    a = np.zeros((2, 2))
    a[1, 0] = 1.0
    return dict(S=2, a=a, b=np.array([0.5, 0.5]), b_err=np.array([-0.5, 0.5]),
                c=np.array([0.0, 1.0]), interp=np.array([[1.0, -0.5], [0.0, 0.5]]),
                order=2, error_order=1, fsal=0)


def _fn(name, values, nidx):
    """A switch-based accessor that folds to an immediate once inlined."""
    lines = [f"BODE_HD_CONSTEXPR double {name}({', '.join('int ' + c for c in 'ij'[:nidx])}) {{"]
    lines.append("  switch (" + ("i * 16 + j" if nidx == 2 else "i") + ") {")
    for idx, v in values:
        if v != 0.0 or np.signbit(v):
            lines.append(f"    case {idx}: return {float(v).hex()}; /* {float(v)!r} */")
    lines.append("    default: return 0.0;")
    lines.append("  }")
    lines.append("}")
    return "\n".join(lines)


def render():
    out = ["/* GENERATED by gen_tableau.py -- do not edit.  Exact binary64 RK tables. */",
           "#pragma once",
           "#if defined(__CUDACC__)",
           "#define BODE_HD_CONSTEXPR __host__ __device__ __forceinline__ constexpr",
           "#elif defined(__cplusplus)",
           "#define BODE_HD_CONSTEXPR inline constexpr",
           "#else",
           "#define BODE_HD_CONSTEXPR static inline",
           "#endif",
           ""]
    for name, t in (("dopri5", dopri5()), ("tsit5", tsit5()), ("heun", heun())):
        S = t["S"]
        out.append(f"/* ---- {name}: stages={S} order={t['order']} error_order={t['error_order']}"
                   f" fsal={t['fsal']} interp_terms={t['interp'].shape[1]} ---- */")
        out.append(f"#define BODE_{name.upper()}_STAGES {S}")
        out.append(f"#define BODE_{name.upper()}_ORDER {t['order']}")
        out.append(f"#define BODE_{name.upper()}_ERROR_ORDER {t['error_order']}")
        out.append(f"#define BODE_{name.upper()}_FSAL {t['fsal']}")
        out.append(f"#define BODE_{name.upper()}_NINTERP {t['interp'].shape[1]}")
        out.append(_fn(f"bode_{name}_a", [(i * 16 + j, t["a"][i, j]) for i in range(S) for j in range(S)], 2))
        out.append(_fn(f"bode_{name}_b", list(enumerate(t["b"])), 1))
        out.append(_fn(f"bode_{name}_berr", list(enumerate(t["b_err"])), 1))
        out.append(_fn(f"bode_{name}_c", list(enumerate(t["c"])), 1))
        out.append(_fn(f"bode_{name}_interp",
                       [(i * 16 + j, t["interp"][i, j]) for i in range(S)
                        for j in range(t["interp"].shape[1])], 2))
        out.append("")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tableau_coeffs.h")
    with open(path, "w") as fh:
        fh.write(render())
    print("wrote", path)
