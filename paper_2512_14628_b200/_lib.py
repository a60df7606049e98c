"""ctypes binding of libhsx.so (include/hsx.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``make``. There
is no fallback: if the shared object is missing or fails to load, every
product entry point raises ``RuntimeError`` naming the build command.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, CudaError, ProtocolError, ShapeError

LIB_PATH = os.environ.get("HSX_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhsx.so")
ABI_VERSION = 1

HSX_OK, HSX_ESHAPE, HSX_EPROTOCOL, HSX_ECONFIG, HSX_ECUDA, HSX_EINVAL = range(6)
SUM_KOUT, SUM_KIN, SUM_ELEMS, SUM_OFFSET, SUM_DRIFT, SUM_POP, SUM_COLS = range(7)
MAX_CONSTRAINTS = 3
RESID_SLOTS = 9     # residual slots per layer (consensus.py:235)

_ERRORS = {HSX_ESHAPE: ShapeError, HSX_EPROTOCOL: ProtocolError, HSX_ECONFIG: ConfigError,
           HSX_ECUDA: CudaError, HSX_EINVAL: ValueError}


class LayerDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("shape", C.c_int32 * 4), ("n_constraints", C.c_int32),
                ("group", C.c_int32 * MAX_CONSTRAINTS), ("keep", C.c_int32 * MAX_CONSTRAINTS),
                ("rho1", C.c_double), ("rho2", C.c_double)]


P, I32, I64, F32, F64, VP = (C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p)


class ResidParams(C.Structure):
    """hsx_resid_params (include/hsx.h)."""
    _fields_ = [("weight_decay", C.c_double), ("eps_abs", C.c_double), ("eps_rel", C.c_double),
                ("mu", C.c_double), ("tau_inc", C.c_double), ("tau_dec", C.c_double),
                ("rho1_max", C.c_double), ("rho2_max", C.c_double),
                ("num_nodes", C.c_int32), ("accels_per_node", C.c_int32), ("adapt", C.c_int32),
                ("flat", C.c_int32)]

# name -> (restype, argtypes); every int-returning entry point is error-checked
SIGNATURES = {
    "hsx_abi_version": (C.c_int, []),
    "hsx_last_error": (C.c_char_p, []),
    "hsx_launch_count": (I64, []),
    "hsx_note_graph_replay": (None, [I64]),
    "hsx_set_l2_hints": (C.c_int, [I32]),
    "hsx_plan_create": (C.c_int, [C.POINTER(LayerDesc), I32, C.POINTER(P)]),
    "hsx_plan_destroy": (None, [P]),
    "hsx_plan_arena_elements": (I64, [P]),
    "hsx_plan_layer_offset": (I64, [P, I32]),
    "hsx_plan_mask_words": (I64, [P]),
    "hsx_plan_mask_word_offset": (I64, [P, I32]),
    "hsx_plan_group_offset": (I64, [P, I32, I32]),
    "hsx_plan_group_total": (I64, [P, I32]),
    "hsx_plan_keep_offset": (I64, [P, I32, I32]),
    "hsx_plan_keep_total": (I64, [P, I32]),
    "hsx_plan_max_passes": (I32, [P]),
    "hsx_plan_set_penalties": (C.c_int, [P, VP, VP, F64, I32, I32, I32]),
    "hsx_pack_theta_u": (C.c_int, [P, VP, VP, VP, VP]),
    "hsx_candidate": (C.c_int, [P, VP, VP, VP, VP, VP, VP, VP, VP]),
    "hsx_candidate_renorm": (C.c_int, [P, I32, VP, VP, VP, VP, VP, VP]),
    "hsx_select": (C.c_int, [P, I32, VP]),
    "hsx_read_groups": (C.c_int, [P, I32, VP, VP, VP]),
    "hsx_project": (C.c_int, [P, VP, VP, VP]),
    "hsx_project_keep_sets": (C.c_int, [P, VP, VP, VP, VP]),
    "hsx_select_project_keep_sets": (C.c_int, [P, VP, VP, VP, VP]),
    "hsx_plan_set_single_node": (C.c_int, [P, C.c_int32]),
    "hsx_plan_set_order": (C.c_int, [P, C.c_int32]),
    "hsx_plan_set_k67_chain": (C.c_int, [P, C.c_int32]),
    "hsx_plan_summary_host": (C.POINTER(C.c_int64), [P]),
    "hsx_mask_or": (C.c_int, [VP, I32, I64, VP, VP]),
    "hsx_keep_sets": (C.c_int, [P, VP, VP, VP]),
    "hsx_keep_sets_fetch": (C.c_int, [P, VP, VP]),
    "hsx_keep_sets_fetch_async": (C.c_int, [P, VP, VP]),
    "hsx_keep_sets_fetch_wait": (C.c_int, [P]),
    "hsx_set_keep_sets": (C.c_int, [P, I32, VP, I32, VP, I32]),
    "hsx_read_keep_positions": (C.c_int, [P, I32, VP, VP]),
    "hsx_compact_dual": (C.c_int, [P, VP, VP, VP, VP, VP, VP]),
    "hsx_dual_intra": (C.c_int, [P, VP, VP, VP, VP]),
    "hsx_decompact_dual": (C.c_int, [P, VP, F32, VP, VP, VP, VP]),
    "hsx_compact_dual_resid": (C.c_int, [P, VP, VP, VP, VP, VP, VP]),
    "hsx_decompact_dual_resid": (C.c_int, [P, VP, F32, VP, VP, VP, VP, VP]),
    "hsx_local_sync": (C.c_int, [P, VP, VP, VP, VP, VP, VP, I32, VP]),
    "hsx_decompact_average": (C.c_int, [P, VP, I32, F64, VP, VP, VP, VP, VP, I32, VP]),
    "hsx_residual_fold": (C.c_int, [P, I32, VP, VP]),
    "hsx_residual_report": (C.c_int, [P, VP, VP, VP, C.POINTER(ResidParams), VP]),
    "hsx_scale_duals": (C.c_int, [P, VP, VP, VP, VP]),
    "hsx_plan_read_penalties": (C.c_int, [P, VP, VP]),
    "hsx_dense_grad_pack": (C.c_int, [VP, VP, F64, VP, C.c_int64, VP]),
    "hsx_dense_apply": (C.c_int, [VP, I32, F64, VP, VP, F64, F64, I32, C.c_int64, VP]),
    "hsx_topk_create": (C.c_int, [VP, VP, F64, I32, VP]),
    "hsx_topk_destroy": (None, [VP]),
    "hsx_topk_total": (I64, [VP]),
    "hsx_topk_layer_keep": (C.c_int, [VP, I32, VP, VP]),
    "hsx_topk_select": (C.c_int, [VP, VP, VP, F64, VP, VP, VP, VP]),
    "hsx_topk_scatter": (C.c_int, [VP, VP, VP, VP, VP]),
    "hsx_topk_apply": (C.c_int, [VP, VP, F64, VP, VP, F64, F64, I32, VP]),
    "hsx_prox_sgd_step": (C.c_int, [P, VP, VP, VP, VP, VP, F64, F64, I32, VP, VP]),
    "hsx_nonzero_u8": (C.c_int, [VP, I64, VP, VP]),
    "hsx_pack_bits": (C.c_int, [VP, I64, VP, VP]),
    "hsx_unpack_bits": (C.c_int, [VP, I64, VP, VP]),
    "hsx_count_diff_u8": (C.c_int, [VP, VP, I64, VP, VP]),
    "hsx_selftest_division": (C.c_int, [VP, I64, F64, VP, VP]),
    "hsx_candidate_peers": (C.c_int, [P, VP, I32, VP, VP, VP, VP, VP]),
    "hsx_plan_set_peer_staging": (C.c_int, [P, I32]),
    "hsx_candidate_peers_staged": (C.c_int, [P, VP, I32, I32, VP, VP, VP, VP, VP]),
    "hsx_mask_or_ptrs": (C.c_int, [VP, I32, I64, VP, VP]),
    "hsx_candidate_renorm_peers": (C.c_int, [P, I32, VP, I32, VP, VP, VP]),
    "hsx_average_peers": (C.c_int, [P, VP, I32, F64, VP, VP]),
    "hsx_group_barrier": (C.c_int, [VP, VP, I32, I32, I32, VP]),
    "hsx_group_barrier_mode": (C.c_int, [VP, VP, I32, I32, I32, I32, I32, VP]),
    "hsx_plan_split_sizes": (C.c_int, [VP, VP, VP]),
    "hsx_keep_sets_ptrs": (C.c_int, [VP, VP, I32, VP, VP, VP]),
    "hsx_candidate_dist": (C.c_int, [VP, VP, I32, VP, VP, VP, VP, VP]),
    "hsx_plan_set_split": (C.c_int, [VP, I32, VP, VP, VP, VP]),
    "hsx_candidate_peers_split": (C.c_int, [VP, VP, I32, VP, VP, VP, VP, VP]),
    "hsx_barrier_timeouts": (C.c_int, [C.POINTER(C.c_uint32), I32]),
    "hsx_slices_peers": (C.c_int, [P, VP, I32, I32, F64, I32, VP, VP]),
}

_lib = None


def load(path: str = LIB_PATH):
    """dlopen libhsx (no CUDA call is made); raises if missing or ABI-mismatched."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"libhsx.so not found at {path}; build it with `make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hsx_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libhsx ABI {lib.hsx_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != HSX_OK:
        msg = load().hsx_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr_array(ptrs):
    """Host array of device pointers (for the *_peers / *_ptrs entry points)."""
    arr = (C.c_void_p * max(len(ptrs), 1))(*[int(p) for p in ptrs])
    return C.cast(arr, C.c_void_p), arr


def launch_count() -> int:
    return int(load().hsx_launch_count())


def barrier_timeouts(reset: bool = False) -> int:
    """Group barriers on the current device that gave up waiting (synchronous)."""
    n = C.c_uint32(0)
    call("hsx_barrier_timeouts", C.byref(n), 1 if reset else 0)
    return int(n.value)


def note_graph_replay(kernels: int) -> None:
    """Count the libhsx kernels of a replayed CUDA graph (captured through this ABI)."""
    load().hsx_note_graph_replay(int(kernels))
