"""ctypes binding of librnndg.so (include/rnndg.h).

There is no fallback: if the CUDA library is missing this module raises, and
every compute entry point needs a visible GPU.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RNNDG_LIB_PATH") or os.path.join(HERE, "librnndg.so")  # override: experiments only

OK, EPARAM, EDATA, EINTERNAL = 0, 1, 2, 3
X_PENDING, X_PROPOSAL, X_INEDGE, X_DELETE = 0, 1, 2, 3

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)


class Counts(C.Structure):
    """rnndg_counts == rnnd::EditCounts (builder.hpp:25-38)."""

    _fields_ = [("removed", C.c_uint64), ("inserted", C.c_uint64),
                ("flag_skips", C.c_uint64), ("pair_checks", C.c_uint64)]


class BuildStatsC(C.Structure):
    _fields_ = [("seconds", C.c_double), ("update_passes", C.c_uint32),
                ("reverse_phases", C.c_uint32), ("edits", Counts),
                ("scan_seconds", C.c_double), ("sort_seconds", C.c_double),
                ("apply_seconds", C.c_double), ("reverse_seconds", C.c_double),
                ("touched", C.c_uint64), ("active_entries", C.c_uint64),
                ("scan_launches", C.c_uint64), ("kernel_launches", C.c_uint64)]


PROGRESS_FN = C.CFUNCTYPE(None, C.c_uint32, C.c_uint32, C.POINTER(Counts), C.c_double,
                          C.c_void_p)

_LIB = None


def lib() -> C.CDLL:
    """Load librnndg.so, raising loudly when the CUDA extension is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "rnndg_create": (C.c_int, [C.POINTER(vp), C.c_int]),
        "rnndg_destroy": (C.c_int, [vp]),
        "rnndg_last_error": (C.c_char_p, [vp]),
        "rnndg_kernel_launches": (C.c_uint64, [vp]),
        "rnndg_set_data": (C.c_int, [vp, f32p, C.c_uint64, C.c_uint32]),
        "rnndg_set_data_device": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32]),
        "rnndg_load_fvecs": (C.c_int, [vp, C.c_char_p, u64p, C.POINTER(C.c_uint32)]),
        "rnndg_random_init": (C.c_int, [vp, C.c_uint32, C.c_uint64]),
        "rnndg_update_pass": (C.c_int, [vp, C.POINTER(Counts)]),
        "rnndg_reverse": (C.c_int, [vp, C.c_uint32, C.c_int]),
        "rnndg_sort_lists": (C.c_int, [vp]),
        "rnndg_build": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.c_uint64, C.c_int, C.POINTER(BuildStatsC),
                                  PROGRESS_FN, vp]),
        "rnndg_pass_counts": (C.c_int, [vp, C.POINTER(Counts), C.c_uint32]),
        "rnndg_graph_size": (C.c_int, [vp, u64p, u64p]),
        "rnndg_get_graph": (C.c_int, [vp, u64p, u32p, f32p, u8p]),
        "rnndg_set_graph": (C.c_int, [vp, C.c_uint64, u64p, u32p, f32p, u8p]),
        "rnndg_index_bytes": (C.c_int, [vp, u8p, u64p]),
        "rnndg_degree_stats": (C.c_int, [vp, C.c_uint32, u64p]),
        "rnndg_search": (C.c_int, [vp, f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                                   C.c_uint64, u32p, f32p, u64p, u64p]),
        "rnndg_brute_force": (C.c_int, [vp, f32p, C.c_uint64, C.c_uint32, u32p]),
        "rnndg_rng_strategy": (C.c_int, [vp, C.c_uint32, u32p, f32p, C.c_uint32, u32p,
                                         f32p, u32p]),
        "rnndg_l2_pairs": (C.c_int, [vp, u32p, u32p, C.c_uint64, f32p]),
        "rnndg_set_partition": (C.c_int, [vp, C.c_uint64, C.c_uint64]),
        "rnndg_shard_scan": (C.c_int, [vp, C.POINTER(Counts), u64p]),
        "rnndg_shard_stage": (C.c_int, [vp, C.c_int, u64p]),
        "rnndg_shard_totals": (C.c_int, [vp, C.POINTER(C.c_double), u64p, u64p, u64p, C.c_int]),
        "rnndg_shard_export": (C.c_int, [vp, u64p, C.c_uint32, vp, vp, u64p]),
        "rnndg_shard_route": (C.c_int, [vp, u64p, C.c_uint32, u64p]),
        "rnndg_shard_push": (C.c_int, [vp, u64p, C.c_uint32, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p), u64p]),
        "rnndg_shard_import": (C.c_int, [vp, C.c_int, vp, vp, C.c_uint64, C.c_uint32,
                                         C.POINTER(Counts), u64p]),
        "rnndg_shard_out_prune": (C.c_int, [vp, C.c_uint32]),
        "rnndg_sharded_create": (C.c_int, [C.POINTER(vp), C.POINTER(C.c_int), C.c_int]),
        "rnndg_sharded_destroy": (C.c_int, [vp]),
        "rnndg_sharded_last_error": (C.c_char_p, [vp]),
        "rnndg_sharded_set_data": (C.c_int, [vp, f32p, C.c_uint64, C.c_uint32]),
        "rnndg_sharded_build": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint64, C.c_int, C.POINTER(BuildStatsC)]),
        "rnndg_sharded_pass_counts": (C.c_int, [vp, C.POINTER(Counts), C.c_uint32,
                                                C.POINTER(C.c_uint32)]),
        "rnndg_sharded_graph_size": (C.c_int, [vp, u64p, u64p]),
        "rnndg_sharded_get_graph": (C.c_int, [vp, u64p, u32p, f32p, u8p]),
        "rnndg_nnd_init": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint64]),
        "rnndg_nnd_pass": (C.c_int, [vp, u64p]),
        "rnndg_nnd_pools": (C.c_int, [vp, u32p, u32p, u32p, f32p, u8p]),
        "rnndg_nnd_finalize": (C.c_int, [vp]),
        "rnndg_nnd_build": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint64, C.POINTER(BuildStatsC)]),
        
        
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def ptr(a, t):
    return a.ctypes.data_as(t)


# every symbol include/rnndg.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "rnndg_create", "rnndg_destroy", "rnndg_last_error", "rnndg_kernel_launches",
    "rnndg_set_data", "rnndg_set_data_device", "rnndg_load_fvecs", "rnndg_random_init",
    "rnndg_update_pass", "rnndg_reverse", "rnndg_sort_lists", "rnndg_build",
    "rnndg_pass_counts", "rnndg_graph_size", "rnndg_get_graph", "rnndg_set_graph",
    "rnndg_index_bytes", "rnndg_degree_stats", "rnndg_search", "rnndg_brute_force",
    "rnndg_rng_strategy", "rnndg_l2_pairs",
    "rnndg_set_partition", "rnndg_shard_scan", "rnndg_shard_stage", "rnndg_shard_export",
    "rnndg_shard_route", "rnndg_shard_push",
    "rnndg_shard_import", "rnndg_shard_out_prune", "rnndg_shard_totals",
    "rnndg_nnd_init", "rnndg_nnd_pass", "rnndg_nnd_pools", "rnndg_nnd_finalize",
    "rnndg_nnd_build",
    "rnndg_sharded_create", "rnndg_sharded_destroy", "rnndg_sharded_last_error",
    "rnndg_sharded_set_data", "rnndg_sharded_build", "rnndg_sharded_pass_counts",
    "rnndg_sharded_graph_size", "rnndg_sharded_get_graph",
)
