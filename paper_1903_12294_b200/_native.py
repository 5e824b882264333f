"""ctypes binding of libmfseg_sm100.so (the C ABI in include/mfseg_sm100.h).

The shared library is built in-tree by `__graft_entry__.build()` (or `make -C
paper_1903_12294_b200/csrc`).  There is no fallback: if the library is
missing, or no CUDA device is present when a kernel is requested, the call
raises.  Device buffers are torch tensors; only raw pointers cross the ABI.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmfseg_sm100.so")

ABI_VERSION = 2
ACC_WORDS = 16
STAT_WORDS = 14
STAT_PARTIAL_WORDS = 18

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double
szt = C.c_size_t


class Params(C.Structure):
    _fields_ = [("k", i32 * 4), ("mins", f64 * 4), ("C", f64 * 4), ("c_f", f64), ("w_d", f64),
                ("w_p", f64), ("w_f", f64), ("eps_c", f64), ("max_iterations", i32),
                ("n_centers", i32)]


class Field(C.Structure):
    _fields_ = [("nx", i32), ("ny", i32), ("nz", i32), ("nt", i32), ("origin", f64 * 3),
                ("spacing", f64 * 3), ("times", vp), ("values", vp), ("offset", i32 * 3)]


class Points(C.Structure):
    _fields_ = [("n", i64), ("xyz", vp), ("t", vp), ("value", vp)]


class Centers(C.Structure):
    _fields_ = [("loc", vp), ("pval", vp), ("fval", vp), ("has_p", vp), ("has_f", vp),
                ("dormant", vp), ("n_points", vp), ("n_fields", vp)]


class Synth(C.Structure):
    _fields_ = [("nx", i32), ("ny", i32), ("nz", i32), ("nt", i32), ("n_traj", i64),
                ("seed", C.c_uint64), ("noise", f64), ("n_blobs", i32), ("dyadic", i32)]


PROGRESS_FN = C.CFUNCTYPE(None, vp, i32, f64)
REDUCE_FN = C.CFUNCTYPE(C.c_int, vp, vp, i64, vp)

P = C.POINTER

_SIGNATURES = {
    "mfseg_last_error": (C.c_char_p, []),
    "mfseg_abi_version": (C.c_int, []),
    "mfseg_launch_count": (C.c_longlong, []),
    "mfseg_set_debug_options": (C.c_int, [i32, i64]),
    "mfseg_timing_enable": (None, [i32]),
    "mfseg_timing_read": (i32, [P(f64), i32]),
    "mfseg_run_workspace_size": (szt, [P(Params), P(Field), P(Points)]),
    "mfseg_run": (C.c_int, [P(Params), P(Field), P(Points), vp, vp, Centers, P(i32), P(i32),
                            PROGRESS_FN, vp, REDUCE_FN, vp, vp, szt, vp]),
    "mfseg_assign_workspace_size": (szt, [P(Params), P(Field), P(Points)]),
    "mfseg_assign": (C.c_int, [P(Params), P(Field), P(Points), Centers, vp, vp, vp, vp, szt, vp]),
    "mfseg_accumulate": (C.c_int, [i32, P(Field), P(Points), vp, vp, vp, vp]),
    "mfseg_acc_to_double": (C.c_int, [i32, vp, vp, vp, vp, vp, vp, vp]),
    "mfseg_update_centers": (C.c_int, [i32, vp, Centers, Centers, f64, P(i32), P(f64), vp]),
    "mfseg_update_centers_f64": (C.c_int, [i32, vp, vp, vp, vp, vp, Centers, Centers, vp]),
    "mfseg_compare_centers": (C.c_int, [i32, Centers, Centers, f64, P(i32), P(f64), vp]),
    "mfseg_minmax_normalize": (C.c_int, [vp, i64, i32, P(f64), P(f64), vp]),
    "mfseg_normalize_range": (C.c_int, [vp, i64, f64, f64, vp]),
    "mfseg_traj_split_workspace_size": (szt, [i64]),
    "mfseg_traj_split": (C.c_int, [i64, vp, vp, vp, vp, vp, P(i64), P(f64), vp, szt, vp]),
    "mfseg_link_index_workspace_size": (szt, [i64]),
    "mfseg_link_index": (C.c_int, [P(Field), P(Points), vp, vp, P(i64), vp, szt, vp]),
    "mfseg_merge_workspace_size": (szt, [i32]),
    "mfseg_merge": (C.c_int, [i32, vp, vp, vp, vp, vp, vp, f64, i32, vp, vp, vp, vp, vp, vp, vp,
                              P(i32), vp, szt, vp]),
    "mfseg_relabel": (C.c_int, [vp, i64, vp, i32, vp, vp]),
    "mfseg_voxel_csr_workspace_size": (szt, [i64, i32, i32]),
    "mfseg_voxel_csr": (C.c_int, [vp, i32, i64, vp, i32, i32, vp, vp, vp, szt, vp]),
    "mfseg_feature_stats_workspace_size": (szt, [i32]),
    "mfseg_feature_stats": (C.c_int, [i32, P(Field), vp, P(Points), vp, vp, vp, szt, vp]),
    "mfseg_traj_split_stride": (C.c_int, [i64, vp, vp, vp, f64, vp, vp, P(i64), vp, szt, vp]),
    "mfseg_feature_stats_pass": (C.c_int, [i32, P(Field), vp, P(Points), vp, i32, vp, vp, vp]),
    "mfseg_feature_stats_means": (C.c_int, [i32, vp, vp, vp]),
    "mfseg_feature_stats_final": (C.c_int, [i32, vp, vp, vp, vp]),
    "mfseg_acc_to_limbs": (C.c_int, [vp, i64, vp, vp]),
    "mfseg_limbs_to_acc": (C.c_int, [vp, i64, vp, vp]),
    "mfseg_synth_field": (C.c_int, [P(Synth), vp, vp]),
    "mfseg_synth_points": (C.c_int, [P(Synth), vp, vp, vp, vp, vp]),
    "mfseg_synth_field_window": (C.c_int, [P(Synth), i32, i32, i32, i32, vp, vp]),
    "mfseg_synth_points_window": (C.c_int, [P(Synth), i64, i64, i32, i32, vp, vp, vp, vp, vp]),
    "mfseg_synth_taxi_points": (C.c_int, [P(Synth), i32, f64, f64, i64, i64, vp, vp, vp, vp, vp]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A call into libmfseg_sm100.so failed; the message is mfseg_last_error()."""


def load():
    """Load the in-tree CUDA library; raise loudly when it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python -c 'import __graft_entry__ as g; g.build()').  There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.mfseg_abi_version() != ABI_VERSION:
            raise ImportError("libmfseg_sm100.so ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().mfseg_last_error().decode(errors="replace")
        if rc == 2:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed (code {rc}): {msg}")


# mfseg_set_debug_options flags (include/mfseg_sm100.h); results never depend on them
DEBUG_NO_CULL = 1
DEBUG_EXACT = 2
DEBUG_STATS = 8
DEBUG_NO_REUSE = 16
DEBUG_NO_MARGIN_REUSE = 32
DEBUG_NO_SEEDS_FAST = 64
DEBUG_NO_ZT_SWAP = 128
DEBUG_NO_BLOCK_CACHE = 256
DEBUG_DEFERRED_BATCH = 512


@contextlib.contextmanager
def debug_options(flags: int = 0, multi_cap: int = -1):
    """Diagnostics / test knobs for library calls made by this thread inside the
    block (the library itself reads no environment variables)."""
    lib = load()
    lib.mfseg_set_debug_options(int(flags), int(multi_cap))
    try:
        yield
    finally:
        lib.mfseg_set_debug_options(0, -1)


def debug_options_from_env() -> None:
    """tools/: map the MFSEG_DEBUG / MFSEG_NO_REUSE / MFSEG_NO_MARGIN_REUSE / MFSEG_NO_SEEDS_FAST /
    MFSEG_MULTI_CAP environment variables onto this thread's debug options."""
    env = os.environ
    flags = int(env.get("MFSEG_DEBUG", "0") or 0)
    flags |= DEBUG_NO_REUSE if env.get("MFSEG_NO_REUSE") else 0
    flags |= DEBUG_NO_MARGIN_REUSE if env.get("MFSEG_NO_MARGIN_REUSE") else 0
    flags |= DEBUG_NO_SEEDS_FAST if env.get("MFSEG_NO_SEEDS_FAST") else 0
    flags |= DEBUG_NO_ZT_SWAP if env.get("MFSEG_NO_ZT_SWAP") else 0
    flags |= DEBUG_NO_BLOCK_CACHE if env.get("MFSEG_NO_BLOCK_CACHE") else 0
    load().mfseg_set_debug_options(flags, int(env.get("MFSEG_MULTI_CAP", "-1")))


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
