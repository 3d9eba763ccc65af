"""Run-time solver specialisations (``bode_program_create``, include/bode.h).

The reference's solve path is open on two sides: any ``ButcherTableau``
(``pkg/src/batchode/tableau.py:17-83``, consumed generically by
``stepper.py:47-110``) and any NumPy dynamics callable
(``stepper.py:19-20``).  libbode's kernels are templates over (tableau,
functor); the built-in pairs are compiled in, any other pair gets its own
specialisation at run time: this module renders the CUDA source (the
tableau's coefficients as compile-time constants, a traced callable as a
device functor -- ``trace.py``) and libbode compiles it with NVRTC for
sm_100a.  Programs are cached per process (and on disk by libbode), keyed
by the generated source, so a dynamics/tableau structure is compiled once
and reused for every batch, parameter value and call.
"""

import ctypes as C
import threading

import numpy as np

from . import _abi

__all__ = ["Program", "get_program", "tableau_source", "dynamics_source"]

SOLVE, STEP, UNITS, JOINT = 1, 2, 4, 8
_BUILTIN_ALIAS = {"vdp": "VdP<O>", "lorenz": "Lorenz<O>", "harmonic": "Harmonic<O>",
                  "damped": "Damped<O>"}


def _lit(v: float) -> str:
    v = float(v)
    if v == 0.0:
        return "-0.0" if np.signbit(v) else "0.0"
    return f"{v.hex()} /* {v!r} */"


def _switch(name, entries, two_d):
    """A constexpr coefficient accessor: switch over the nonzero entries."""
    args = "int i, int j" if two_d else "int i"
    key = "i * 64 + j" if two_d else "i"
    cases = "\n".join(f"    case {k}: return {_lit(v)};" for k, v in entries if v != 0.0)
    return (f"__host__ __device__ __forceinline__ constexpr double {name}({args}) {{\n"
            f"  switch ({key}) {{\n{cases}\n    default: return 0.0;\n  }}\n}}\n")


def tableau_source(tab) -> str:
    """``TabShape<3>`` / ``Tab<3>`` (BODE_METHOD_CUSTOM) for a user tableau:
    the same accessors the built-in tableaus have (bode_device.cuh), with
    every coefficient a compile-time constant, so zero terms fold away
    exactly as for dopri5 / tsit5."""
    S = int(tab.stages)
    a, b, e, c = (np.asarray(x, dtype=np.float64) for x in (tab.a, tab.b, tab.b_err, tab.c))
    w = np.asarray(tab.interp_coeffs, dtype=np.float64)
    if w.ndim != 2 or w.shape[0] != S or w.shape[1] < 1:
        raise ValueError("interp_coeffs must be (stages, m) with m >= 1")
    NI = w.shape[1]
    fns = (_switch("user_a", [(i * 64 + j, a[i, j]) for i in range(S) for j in range(S)], True)
           + _switch("user_b", list(enumerate(b)), False)
           + _switch("user_e", list(enumerate(e)), False)
           + _switch("user_c", list(enumerate(c)), False)
           + _switch("user_w", [(i * 64 + j, w[i, j]) for i in range(S) for j in range(NI)],
                     True))
    acc = ("  static __device__ __forceinline__ constexpr double za(int i, int j) { return user_a(i, j); }\n"
           "  static __device__ __forceinline__ constexpr double zb(int i) { return user_b(i); }\n"
           "  static __device__ __forceinline__ constexpr double ze(int i) { return user_e(i); }\n"
           "  static __device__ __forceinline__ constexpr double zw(int i, int j) { return user_w(i, j); }\n")
    return f"""namespace bode {{
// user ButcherTableau (tableau.py:17-83): stages={S} order={tab.order} error_order={tab.error_order} fsal={bool(tab.fsal)}
{fns}
template <> struct TabShape<BODE_METHOD_CUSTOM> {{
  static constexpr int S = {S}, ORDER = {int(tab.order)}, ERR_ORDER = {int(tab.error_order)}, NI = {NI};
  static constexpr bool FSAL = {"true" if tab.fsal else "false"};
{acc}}};
template <> struct Tab<BODE_METHOD_CUSTOM> : TabShape<BODE_METHOD_CUSTOM> {{
  static __device__ __forceinline__ double a(int i, int j) {{ return user_a(i, j); }}
  static __device__ __forceinline__ double b(int i) {{ return user_b(i); }}
  static __device__ __forceinline__ double e(int i) {{ return user_e(i); }}
  static __device__ __forceinline__ double c(int i) {{ return user_c(i); }}
  static __device__ __forceinline__ double w(int i, int j) {{ return user_w(i, j); }}
}};
}}  // namespace bode
"""


def dynamics_source(dyn, d: int) -> str:
    """``UserDyn<O>`` for a registered functor (an alias) or a traced one."""
    if getattr(dyn, "kind", None) == "program":
        return dyn.traced.source
    if dyn.kind == "mlp":
        raise NotImplementedError("MLP dynamics run on the fused tcgen05 kernel; they do not "
                                  "combine with a custom tableau or the stepping API")
    alias = _BUILTIN_ALIAS.get(dyn.kind, f"Elementwise<O, {d}>")
    return f"namespace bode {{\ntemplate <class O>\nusing UserDyn = {alias};\n}}  // namespace bode\n"


class Program:
    """A compiled specialisation (owns the ``bode_program*``)."""

    def __init__(self, ptr, desc):
        self.ptr, self.desc = ptr, desc

    @property
    def handle(self):
        return self.ptr.value



# Programs live for the process: a solve launched with one may still be
# running when its Python references are gone, and there are only as many
# programs as distinct (tableau, dynamics) structures.
_cache = {}
_retired = []
_lock = threading.Lock()


def get_program(method, dyn, d: int, kernels: int) -> Program:
    """The program for (method, dynamics, width) with at least ``kernels``.
    ``method``: a built-in name or a custom ``ButcherTableau``."""
    lib = _abi.load()
    custom = not isinstance(method, str)
    src = (tableau_source(method) if custom else "") + dynamics_source(dyn, d)
    mid = _abi.METHOD_CUSTOM if custom else _abi.METHOD[method]
    import torch
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    n_params = dyn.n_params if getattr(dyn, "kind", None) == "program" else 0
    key = (src, mid, d, n_params, dev)
    with _lock:
        have = _cache.get(key)
        if have is not None and (have.desc.kernels & kernels) == kernels:
            return have
        want = kernels | (have.desc.kernels if have is not None else 0)
        desc = _abi.ProgramDesc()
        desc.method, desc.kernels, desc.d, desc.n_params = mid, want, d, n_params
        if custom:
            desc.stages, desc.order = int(method.stages), int(method.order)
            desc.error_order, desc.fsal = int(method.error_order), int(bool(method.fsal))
        else:
            desc.stages = 2 if method == "heun" else 7
            desc.order = 2 if method == "heun" else 5
            desc.error_order = 1 if method == "heun" else 4
            desc.fsal = 0 if method == "heun" else 1
        ptr = C.c_void_p()
        _abi.check(lib.bode_program_create(src.encode(), C.byref(desc), C.byref(ptr)))
        prog = Program(ptr, desc)
        if have is not None:
            _retired.append(have)
        _cache[key] = prog
        return prog
