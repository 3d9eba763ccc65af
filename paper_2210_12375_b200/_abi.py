"""ctypes binding of ``libbode.so`` (the C ABI declared in include/bode.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2210_12375_b200/csrc``) into ``paper_2210_12375_b200/_build``.
There is deliberately no fallback: if the CUDA library is missing, every
solve raises ``BodeLibraryError``.
"""

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BODE_LIB") or os.path.join(HERE, "_build", "libbode.so")

ABI_VERSION = 6
TRAJ_EXTRA = 3


def mlp_stage_record(a) -> int:
    """Stages per recorded step of the fp32 stage-input record the
    tensor-core MLP backward needs (bode_solve_args.traj_stages): the fused
    integrator's shapes (d == 64, hidden a multiple of 32 up to 256), built-in
    tableaus; 0 otherwise."""
    if a.dyn.kind != DYN["mlp"] or a.d != 64 or a.program:
        return 0
    h = a.dyn.hidden
    if h % 32 or not 32 <= h <= 256:
        return 0
    return STAGES.get(a.method, 0)


def traj_stride(d: int) -> int:
    """BODE_TRAJ_STRIDE(d): doubles per recorded accepted step."""
    return (d + TRAJ_EXTRA + 3) // 4 * 4
OK, EINVAL, ECUDA, EUNSUPPORTED = 0, 1, 2, 3
METHOD = {"dopri5": 0, "tsit5": 1, "heun": 2}
METHOD_CUSTOM = 3
STAGES = {0: 7, 1: 7, 2: 2}  # per METHOD value
MODE = {"exact": 0, "fast": 1}
DT0_HEURISTIC, DT0_SCALAR, DT0_ARRAY = 0, 1, 2
DYN = {"vdp": 1, "lorenz": 2, "zero": 3, "const": 4, "linear": 5, "linear_cos": 6,
       "linear_sin": 7, "relax_cos": 8, "square": 9, "logistic": 10, "sin_plus_t": 11,
       "harmonic": 12, "damped": 13, "mlp": 20, "program": 30}


class BodeLibraryError(RuntimeError):
    """libbode.so is missing or failed (CUDA error)."""


class Dynamics_(C.Structure):
    _fields_ = [("kind", C.c_int32), ("inst_mask", C.c_uint32),
                ("inst_params", C.c_void_p), ("shared_params", C.c_double * 8),
                ("W1", C.c_void_p), ("b1", C.c_void_p), ("W2", C.c_void_p),
                ("b2", C.c_void_p), ("hidden", C.c_int64)]


class Controller_(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("beta3", C.c_double),
                ("safety", C.c_double), ("factor_min", C.c_double),
                ("factor_max", C.c_double), ("update_history_on_reject", C.c_int32),
                ("_pad", C.c_int32)]


class SolveArgs(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("method", C.c_int32), ("mode", C.c_int32),
                ("dt0_mode", C.c_int32), ("n", C.c_int64), ("d", C.c_int64),
                ("dyn", Dynamics_), ("ctrl", Controller_),
                ("y0", C.c_void_p), ("t_start", C.c_void_p), ("t_end", C.c_void_p),
                ("t_eval", C.c_void_p), ("t_eval_offsets", C.c_void_p),
                ("t_eval_len", C.c_int64), ("atol_v", C.c_void_p), ("rtol_v", C.c_void_p),
                ("atol", C.c_double), ("rtol", C.c_double), ("max_steps", C.c_int64),
                ("dt0", C.c_double), ("dt0_v", C.c_void_p), ("order", C.c_void_p),
                ("ys", C.c_void_p), ("n_emitted", C.c_void_p), ("n_steps", C.c_void_p),
                ("n_accepted", C.c_void_p), ("final_dt", C.c_void_p),
                ("status", C.c_void_p), ("n_f_evals", C.c_void_p),
                ("trace_t", C.c_void_p), ("trace_dt", C.c_void_p),
                ("trace_accept", C.c_void_p), ("trace_cap", C.c_int64),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("stream", C.c_void_p), ("threads_per_block", C.c_int32),
                ("blocks", C.c_int32), ("cost_hint", C.c_void_p),
                ("pipeline_chunks", C.c_int32), ("joint", C.c_int32),
                ("max_iterations_out", C.c_void_p), ("refresh_map_out", C.c_void_p),
                ("reserved_mlp", C.c_int32), ("_pad3", C.c_int32),
                ("prof_event_start", C.c_void_p), ("prof_event_stop", C.c_void_p),
                ("launch_count_out", C.c_void_p),
                ("traj", C.c_void_p), ("traj_offsets", C.c_void_p),
                ("program", C.c_void_p), ("traj_stages", C.c_void_p)]


class ProgramDesc(C.Structure):
    _fields_ = [("method", C.c_int32), ("kernels", C.c_int32), ("d", C.c_int64),
                ("n_params", C.c_int32), ("stages", C.c_int32), ("order", C.c_int32),
                ("error_order", C.c_int32), ("fsal", C.c_int32), ("_pad", C.c_int32)]


TAB_MAX_STAGES, TAB_MAX_INTERP = 16, 8


class Tableau_(C.Structure):
    _fields_ = [("stages", C.c_int32), ("n_interp", C.c_int32), ("fsal", C.c_int32),
                ("_pad", C.c_int32), ("a", C.c_double * (TAB_MAX_STAGES * TAB_MAX_STAGES)),
                ("b", C.c_double * TAB_MAX_STAGES), ("b_err", C.c_double * TAB_MAX_STAGES),
                ("c", C.c_double * TAB_MAX_STAGES),
                ("interp", C.c_double * (TAB_MAX_STAGES * TAB_MAX_INTERP))]


class StepState(C.Structure):
    _fields_ = [("t", C.c_void_p), ("y", C.c_void_p), ("f0", C.c_void_p),
                ("norm_prev", C.c_void_p), ("norm_prev2", C.c_void_p), ("te_next", C.c_void_p),
                ("fsal_valid", C.c_void_p), ("flags", C.c_void_p)]


class AdjointArgs(C.Structure):
    _fields_ = [("traj", C.c_void_p), ("traj_offsets", C.c_void_p),
                ("n_emitted", C.c_void_p), ("grad_ys", C.c_void_p),
                ("grad_y0", C.c_void_p), ("grad_params", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("launch_count_out", C.c_void_p), ("grad_W1", C.c_void_p),
                ("grad_b1", C.c_void_p), ("grad_W2", C.c_void_p), ("grad_b2", C.c_void_p),
                ("traj_stages", C.c_void_p)]


# every symbol include/bode.h declares, with its ctypes signature
_P, _I32, _I64, _D, _SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
SIGNATURES = {
    "bode_abi_version": ([], C.c_int),
    "bode_sizeof_args": ([], _SZ),
    "bode_last_error": ([], C.c_char_p),
    "bode_workspace_size": ([C.POINTER(SolveArgs)], _SZ),
    "bode_solve": ([C.POINTER(SolveArgs)], C.c_int),
    "bode_solve_host": ([C.POINTER(SolveArgs)], C.c_int),
    "bode_adjoint_workspace_size": ([C.POINTER(SolveArgs)], _SZ),
    "bode_solve_adjoint": ([C.POINTER(SolveArgs), C.POINTER(AdjointArgs)], C.c_int),
    "bode_rk_step": ([_I32, _I32, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "bode_interpolate": ([_I32, _I32, _I64, _I64, _P, _P, _P, _P, _P, _P], C.c_int),
    "bode_error_norm": ([_I64, _I64, _P, _P, _P, _P, _P, _D, _D, _P, _P], C.c_int),
    "bode_adapt_step": ([_I64, _P, _I32, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "bode_initial_step": ([_P, _I64, _I64, _P, _P, _I32, _P, _P, _D, _D, _P, _P, _P, _P],
                          C.c_int),
    "bode_probe_fp64": ([_I64, _I32, _P, _P], C.c_int),
    "bode_eval_dynamics": ([_P, _I64, _I64, _P, _P, _P, _P], C.c_int),
    "bode_partition_workspace_size": ([_I64], _SZ),
    "bode_program_create": ([C.c_char_p, _P, _P], C.c_int),
    "bode_program_check": ([C.c_char_p, _P], C.c_int),
    "bode_program_destroy": ([_P], None),
    "bode_step_begin": ([C.POINTER(SolveArgs), _P], C.c_int),
    "bode_step_once": ([C.POINTER(SolveArgs), _P], C.c_int),
    "bode_program_rk_step": ([_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "bode_interpolate_tab": ([_P, _I64, _I64, _P, _P, _P, _P, _P, _P], C.c_int),
    "bode_program_initial_step": ([_P, _P, _I64, _I64, _P, _P, _I32, _P, _P, _D, _D, _P, _P,
                                   _P, _P], C.c_int),
    "bode_partition": ([_P, _I64, _I32, _P, _P, _P, _SZ, _P], C.c_int),
    "bode_probe_tf32": ([_I32, _I32, _P], C.c_int),
    "bode_solve_multi": ([C.POINTER(SolveArgs), _I32, _P], C.c_int),
}

_lib = None


def load():
    """Load libbode.so once; raises BodeLibraryError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BodeLibraryError(
            f"{LIB_PATH} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.bode_abi_version() != ABI_VERSION:
        raise BodeLibraryError("libbode.so ABI version mismatch")
    if lib.bode_sizeof_args() != C.sizeof(SolveArgs):
        raise BodeLibraryError("bode_solve_args layout mismatch between header and binding")
    _lib = lib
    return lib


def check(rc):
    """Map a C return code onto the reference's exception types."""
    if rc == OK:
        return
    msg = load().bode_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise BodeLibraryError(msg)
