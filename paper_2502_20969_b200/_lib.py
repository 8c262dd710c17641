"""ctypes binding of liblaivg.so (include/laivg.h).

Loads the in-tree library and fails loudly when it is missing: there is no
CPU or PyTorch fallback for the device path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblaivg.so")

OK, EINVAL, ERUNTIME, ELOGIC, ECUDA = 0, -1, -2, -3, -4


class LogicError(RuntimeError):
    """std::logic_error analogue (double insert, evicting a non-resident cluster)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the library."""


u32, u64, i32, f32, f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_double
vp = C.c_void_p
P = C.POINTER


class Opts(C.Structure):
    _fields_ = [("device", i32), ("capacity_bytes", u64), ("miss_threads", u32),
                ("max_batch", u32), ("max_probe", u32), ("acc_fp64", u32),
                ("scan_impl", u32), ("tma_tile", u32), ("tma_stages", u32),
                ("ctas_per_sm", u32), ("coarse_impl", u32), ("miss_fetch", u32),
                ("fetch_chunk_mb", u32), ("single_chain", u32)]


class Channel(C.Structure):
    _fields_ = [("bandwidth_bytes_per_s", f64), ("mode", i32)]


class TransferReportC(C.Structure):
    _fields_ = [("t_p", f64), ("bytes", u64), ("overshoot_s", f64), ("n_transferred", u32),
                ("window_s", f64), ("h2d_gbps", f64), ("window_read_gbps", f64)]


class CostModelC(C.Structure):
    _fields_ = [("bandwidth_bytes_per_s", f64), ("t_cc", f64), ("t_gc", f64),
                ("parallel_slots", i32)]


class HybridTimingC(C.Structure):
    _fields_ = [("t_g", f64), ("t_c", f64), ("t_2", f64), ("model_t_g", f64),
                ("model_t_c", f64), ("model_t_2", f64), ("t_coarse", f64), ("t_scan", f64),
                ("scanned_vectors", u64), ("scanned_bytes", u64), ("fetched_lists", u32),
                ("cpu_lists", u32), ("fetched_bytes", u64), ("t_fetch", f64),
                ("peer_lists", u32), ("list_scan", u32), ("peer_bytes", u64),
                ("h2d_bytes", u64), ("d2h_bytes", u64), ("t_kernel", f64),
                ("distinct_bytes", u64)]


# name -> (restype, argtypes); every symbol declared in include/laivg.h
SIGNATURES = {
    "laivg_last_error": (C.c_char_p, []),
    "laivg_version": (u32, []),
    "laivg_host_alloc": (i32, [u64, P(vp)]),
    "laivg_host_free": (i32, [vp]),
    "laivg_host_register": (i32, [vp, u64]),
    "laivg_host_unregister": (i32, [vp]),
    "laivg_kernel_launches": (u64, []),
    "laivg_index_create": (i32, [vp, u32, u32, i32, vp, vp, vp, u32, P(vp)]),
    "laivg_index_destroy": (None, [vp]),
    "laivg_index_load": (i32, [C.c_char_p, u32, P(vp)]),
    "laivg_index_save": (i32, [vp, C.c_char_p, u32]),
    "laivg_index_store": (i32, [vp, P(vp), P(vp), P(vp), P(vp)]),
    "laivg_index_num_clusters": (u32, [vp]),
    "laivg_index_dim": (u32, [vp]),
    "laivg_index_metric": (i32, [vp]),
    "laivg_index_total_vectors": (u64, [vp]),
    "laivg_index_cluster_bytes": (u64, [vp, u32]),
    "laivg_index_total_payload_bytes": (u64, [vp]),
    "laivg_index_list_len": (u64, [vp, u32]),
    "laivg_score_clusters": (i32, [vp, vp, vp, u32, u64, vp, vp, P(u64)]),
    "laivg_exact_search": (i32, [vp, vp, u32, i32, vp, vp, vp]),
    "laivg_pairwise_l2": (i32, [vp, vp, u64, vp, u64, u32, vp]),
    "laivg_opts_default": (None, [P(Opts)]),
    "laivg_ctx_create": (i32, [vp, P(Opts), P(vp)]),
    "laivg_ctx_destroy": (None, [vp]),
    "laivg_ctx_sync": (i32, [vp]),
    "laivg_rank_clusters": (i32, [vp, vp, u32, vp, vp]),
    "laivg_coarse_probe": (i32, [vp, vp, u32, i32, vp, P(u32)]),
    "laivg_search_clusters": (i32, [vp, vp, vp, u32, i32, vp, vp, P(u32)]),
    "laivg_ivf_search": (i32, [vp, vp, u32, i32, i32, vp, vp, vp]),
    "laivg_store_capacity_bytes": (u64, [vp]),
    "laivg_store_used_bytes": (u64, [vp]),
    "laivg_store_free_bytes": (u64, [vp]),
    "laivg_store_contains": (i32, [vp, u32]),
    "laivg_store_resident_count": (u32, [vp]),
    "laivg_store_resident": (i32, [vp, vp, vp, vp, P(u32)]),
    "laivg_store_insert": (i32, [vp, u32, i32]),
    "laivg_store_evict": (i32, [vp, u32, P(u64)]),
    "laivg_store_retag_all": (i32, [vp, i32]),
    "laivg_store_clear": (i32, [vp]),
    "laivg_store_bytes_with_tag": (u64, [vp, i32]),
    "laivg_store_recompute_used_bytes": (u64, [vp]),
    "laivg_store_compact": (i32, [vp]),
    "laivg_plan_prefetch": (i32, [vp, vp, u64, vp, P(u32), P(u64), vp, P(u32)]),
    "laivg_execute_prefetch": (i32, [vp, vp, u32, P(Channel), f64, vp, P(TransferReportC)]),
    "laivg_incremental_prefetch": (i32, [vp, vp, u64, P(Channel), f64, vp,
                                         P(TransferReportC)]),
    "laivg_window": (i32, [vp, f64, P(f64)]),
    "laivg_window_load": (i32, [vp, u64, f64]),
    "laivg_link_peak": (i32, [vp, u64, P(f64), P(f64)]),
    "laivg_link_bytes": (i32, [vp, P(u64), P(u64)]),
    "laivg_list_scan_stats": (i32, [vp, P(u64), P(u64), P(f64)]),
    "laivg_hybrid_search": (i32, [vp, vp, i32, i32, P(CostModelC), vp, vp, P(u32), vp,
                                  P(u32), vp, P(u32), P(f64), P(HybridTimingC)]),
    "laivg_coverage": (i32, [vp, vp, vp, i32, P(f64)]),
    "laivg_stage_queries": (i32, [vp, vp, u32]),
    "laivg_hybrid_search_staged": (i32, [vp, u32, i32, i32, vp, vp, P(u32), P(u32),
                                         P(HybridTimingC)]),
    "laivg_hybrid_search_batch": (i32, [vp, vp, u32, i32, i32, vp, vp, vp, vp, vp,
                                        P(HybridTimingC)]),
    "laivg_hybrid_search_batch_staged": (i32, [vp, u32, u32, i32, i32, vp, vp, vp, vp,
                                               P(HybridTimingC)]),
    "laivg_debug_coarse_approx": (i32, [vp, vp, u32, vp]),
    "laivg_synth_queries_topical": (i32, [u64, vp, u32, vp, vp, u32, u32, f64, u32, u32, f32,
                                          vp, vp, vp, vp]),
    "laivg_prefetch_batch": (i32, [vp, vp, u32, vp, P(Channel), f64, vp, vp,
                                   P(TransferReportC)]),
    "laivg_group_microbatches": (i32, [vp, u64, u32, u64, vp, vp, P(u32)]),
    "laivg_slow_tier_scan": (i32, [vp, vp, u32, vp, vp, i32, u32, vp, vp, vp]),
    "laivg_epoch_open": (i32, [vp]),
    "laivg_epoch_close": (i32, [vp]),
    "laivg_store_offsets": (i32, [vp, vp]),
    "laivg_slab_ipc_handle": (i32, [vp, vp]),
    "laivg_peer_attach_ipc": (i32, [vp, u32, vp]),
    "laivg_peer_attach_local": (i32, [vp, u32, vp]),
    "laivg_peer_publish": (i32, [vp, u32, vp]),
    "laivg_group_microbatches_gpu": (i32, [vp, vp, u64, u64, vp, vp, P(u32)]),
    "laivg_schedule": (i32, [vp, vp, u64, u64, i32, vp, u32, vp, vp, P(u32), vp, vp]),
    "laivg_chunk_microbatches": (i32, [u64, u64, vp, vp, P(u32)]),
    "laivg_assign_cache_aware": (i32, [vp, vp, vp, u32, vp, u32, vp, u64, i32, vp]),
    "laivg_greedy_assign": (i32, [vp, u32, u32, vp]),
    "laivg_assign_round_robin": (i32, [u64, u64, vp]),
    "laivg_assignment_overlap": (i32, [vp, vp, vp, u32, vp, u32, vp, vp, u64, i32, P(u64)]),
    "laivg_split_budget": (i32, [u64, vp, u64, vp]),
    "laivg_hotness_create": (i32, [f32, f32, f32, f64, P(vp)]),
    "laivg_hotness_destroy": (None, [vp]),
    "laivg_hotness_on_fetch": (i32, [vp, u32]),
    "laivg_hotness_end_of_round": (i32, [vp, vp, u32]),
    "laivg_hotness_evict_to_fraction": (i32, [vp, vp, vp, P(u32)]),
    "laivg_hotness_get": (f32, [vp, u32]),
    "laivg_hotness_forget": (i32, [vp, u32]),
    "laivg_hotness_clear": (i32, [vp]),
    "laivg_synth_centroids": (i32, [u64, u32, u32, vp]),
    "laivg_synth_lists": (i32, [u64, vp, u32, u32, u64, f32, u32, u32, vp, vp, i32]),
    "laivg_synth_queries": (i32, [u64, vp, u64, u32, u32, f32, vp, vp, vp]),
}

_lib = None


def lib():
    """The loaded library (loads once). Raises ImportError when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2502_20969_b200.build` "
                "(there is no fallback implementation)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().laivg_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ELOGIC:
        raise LogicError(msg)
    if rc == ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)
