"""Embedded Runge-Kutta pairs (host-side data, reference API mirror).

Mirrors ``batchode.tableau`` (reference ``pkg/src/batchode/tableau.py``):
``ButcherTableau`` (:17-57) with ``validate`` (:59-83), ``dopri5`` (:102-149)
and ``tsit5`` (:152-254, interpolant expanded with ``np.polymul`` as
:86-99 does), plus the Heun-Euler pair the torchode API names (SURVEY.md
§8(b)).  The device kernels do not read these arrays at run time: the same
values are compiled in from ``csrc/tableau_coeffs.h``, which
``csrc/gen_tableau.py`` renders from the functions below; a test checks
the committed header, these arrays and the reference tables agree bit for
bit.  Any other (validated) tableau runs through a run-time specialisation
of the same kernels with its coefficients compiled in (program.py).
"""

import functools
from dataclasses import dataclass

import numpy as np

__all__ = ["ButcherTableau", "dopri5", "tsit5", "heun"]


@dataclass(frozen=True, eq=False)
class ButcherTableau:
    stages: int
    a: np.ndarray
    b: np.ndarray
    b_err: np.ndarray
    c: np.ndarray
    order: int
    error_order: int
    interp_coeffs: np.ndarray
    fsal: bool
    method: str = ""

    def validate(self, tol: float = 1e-12) -> None:
        """Consistency checks of tableau.py:59-83 (row sums, quadrature,
        interpolant endpoint, FSAL structure); raises ValueError."""
        if self.a.shape != (self.stages, self.stages):
            raise ValueError("a must be (stages, stages)")
        if np.any(np.triu(self.a) != 0.0):
            raise ValueError("a must be strictly lower triangular")
        if np.max(np.abs(self.a.sum(axis=1) - self.c)) > tol:
            raise ValueError("stage row sums must equal c")
        if abs(self.b.sum() - 1.0) > tol:
            raise ValueError("solution weights must sum to 1")
        if abs(self.b_err.sum()) > tol:
            raise ValueError("error weights must sum to 0")
        if np.max(np.abs(self.interp_coeffs.sum(axis=1) - self.b)) > tol:
            raise ValueError("interpolant at theta=1 must reproduce b")
        if self.fsal and (self.c[-1] != 1.0 or np.max(np.abs(self.a[-1] - self.b)) > tol):
            raise ValueError("fsal requires c[-1] = 1 and a[-1] = b")


def _make(method, t):
    return ButcherTableau(stages=t["S"], a=t["a"], b=t["b"], b_err=t["b_err"], c=t["c"],
                          order=t["order"], error_order=t["error_order"],
                          interp_coeffs=t["interp"], fsal=bool(t["fsal"]), method=method)


def _dopri5_data():
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


def _tsit5_data():
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


def _heun_data():
    a = np.zeros((2, 2))
    a[1, 0] = 1.0
    return dict(S=2, a=a, b=np.array([0.5, 0.5]), b_err=np.array([-0.5, 0.5]),
                c=np.array([0.0, 1.0]), interp=np.array([[1.0, -0.5], [0.0, 0.5]]),
                order=2, error_order=1, fsal=0)


def dopri5() -> ButcherTableau:
    """Dormand-Prince 5(4) with Shampine's dense output (tableau.py:102-149)."""
    return _make("dopri5", _dopri5_data())


def tsit5() -> ButcherTableau:
    """Tsitouras 5(4) with its published interpolant (tableau.py:152-254)."""
    return _make("tsit5", _tsit5_data())


def heun() -> ButcherTableau:
    """Heun-Euler 2(1), non-FSAL, quadratic dense output."""
    return _make("heun", _heun_data())


@functools.lru_cache(maxsize=1)
def _builtin_refs():
    """The built-in pairs, constructed (and validated) once per process, not
    on every solve() call."""
    return (("dopri5", dopri5()), ("tsit5", tsit5()), ("heun", heun()))


def method_of(tableau):
    """Device method for a tableau: the name of a built-in pair (compiled
    into libbode) when the coefficients equal one -- whatever object carries
    them, e.g. a reference-built ``batchode.dopri5()`` -- else the validated
    tableau itself, which runs through a run-time program (program.py)."""
    if tableau is None:
        return "dopri5"
    if isinstance(tableau, str):
        if tableau not in ("dopri5", "tsit5", "heun"):
            raise ValueError(f"unknown method {tableau!r}")
        return tableau
    for k in ("stages", "a", "b", "b_err", "c", "order", "error_order", "interp_coeffs", "fsal"):
        if not hasattr(tableau, k):
            raise TypeError(f"tableau has no {k!r}: expected a ButcherTableau")
    for name, ref in _builtin_refs():
        if int(tableau.stages) == ref.stages and bool(tableau.fsal) == ref.fsal and \
                int(tableau.order) == ref.order and int(tableau.error_order) == ref.error_order and \
                all(np.array_equal(np.asarray(getattr(tableau, k), dtype=np.float64),
                                   getattr(ref, k))
                    for k in ("a", "b", "b_err", "c", "interp_coeffs")):
            return name
    S = int(tableau.stages)
    if S < 1 or S > 16 or np.shape(tableau.interp_coeffs)[1] > 8:
        raise NotImplementedError("device tableaus: at most 16 stages and 8 interpolant terms")
    return tableau


def is_custom(method) -> bool:
    return not isinstance(method, str)


def stages_of(method) -> int:
    return int(method.stages) if is_custom(method) else (2 if method == "heun" else 7)


def fsal_of(method) -> bool:
    return bool(method.fsal) if is_custom(method) else method != "heun"


def order_of(method) -> int:
    return int(method.order) if is_custom(method) else (2 if method == "heun" else 5)


def error_order_of(method) -> int:
    return int(method.error_order) if is_custom(method) else (1 if method == "heun" else 4)
