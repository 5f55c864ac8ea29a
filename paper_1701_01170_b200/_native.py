"""ctypes binding of libgfx.so (include/gfx.h).

This is the only place Python touches the native library.  There is no CPU
fallback: if the shared library is missing or no CUDA device is visible, the
primitives raise instead of silently computing something else.
"""
from __future__ import annotations

import ctypes
import os
import threading
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int, c_int32,
                    c_int64, c_uint64, c_void_p)
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libgfx.so"

GFX_OK, GFX_EINVAL, GFX_ECUDA, GFX_ENOMEM, GFX_ENCCL = range(5)
UNVISITED32 = 2147483647
GRAPH_UNDIRECTED = 1
DIR_PUSH, DIR_PULL, DIR_AUTO = 0, 1, 2
FILTER_EXACT, FILTER_INEXACT = 0, 1
LOOP_HOST, LOOP_DEVICE = 0, 1

(FN_NONE, FN_BFS_CLAIM, FN_BFS_IDEMP, FN_SSSP_RELAX, FN_TC_ORIENT, FN_LABEL_EQ, FN_LABEL_NE,
 FN_SET_LABEL, FN_ADD_I64, FN_BFS_PULL, FN_BC_CLAIM, FN_BC_SIGMA, FN_BC_DELTA, FN_PR_SCATTER,
 FN_PR_MOVED, FN_CC_SAME_COMP, FN_SSSP_STAMP) = range(17)
KIND_V2V, KIND_V2E, KIND_E2V, KIND_E2E = range(4)


class IterRec(Structure):
    _fields_ = [
        ("iteration", c_int64), ("frontier_in", c_int64), ("frontier_out", c_int64),
        ("n_u", c_int64), ("edges", c_int64), ("m_f", c_double), ("m_u", c_double),
        ("mode_before", c_int32), ("decision", c_int32), ("ms", c_float), ("pad", c_int32),
        ("candidates", c_int64), ("work", c_int64), ("bytes_alg", c_int64),
    ]


class Stats(Structure):
    _fields_ = [
        ("iterations", c_int64), ("edges_traversed", c_int64),
        ("direction_switches", c_int64), ("reached", c_int64), ("edges_reached", c_int64),
        ("work_slots", c_int64), ("bytes_alg", c_int64), ("device_ms", c_double),
        ("num_records", c_int64), ("init_ns", c_int64), ("loop_ns", c_int64),
    ]


DBFS_CB0 = ctypes.CFUNCTYPE(c_int, c_void_p)
DBFS_CB_PAIRS = ctypes.CFUNCTYPE(c_int, c_void_p, POINTER(c_int64), POINTER(c_int64))


class DbfsComm(Structure):
    """gfx_dbfs_comm: the collective table of gfx_dbfs_run_comm."""
    _fields_ = [("user", c_void_p), ("exchange_counts", DBFS_CB0),
                ("exchange_pairs", DBFS_CB_PAIRS), ("allgather_frontier", DBFS_CB0),
                ("allreduce_stats", DBFS_CB0)]


class FunctorArgs(Structure):
    _fields_ = [("labels_d", c_void_p), ("preds_d", c_void_p), ("value", c_int64),
                ("f0_d", c_void_p), ("f1_d", c_void_p), ("scalar", c_double)]


# name -> (restype, argtypes); every function listed here is declared in gfx.h
_SIGS = {
    "gfx_version": (c_int, []),
    "gfx_launch_count": (c_int64, []),
    "gfx_ctx_set_timing": (c_int, [c_void_p, c_int]),
    "gfx_ctx_set_stats": (c_int, [c_void_p, c_int]),
    "gfx_last_error": (c_char_p, []),
    "gfx_ctx_create": (c_int, [c_int, c_void_p, POINTER(c_void_p)]),
    "gfx_ctx_destroy": (c_int, [c_void_p]),
    "gfx_ctx_sync": (c_int, [c_void_p]),
    "gfx_ctx_sm_count": (c_int, [c_void_p]),
    "gfx_graph_create": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                 c_int, POINTER(c_void_p)]),
    "gfx_graph_set_reverse": (c_int, [c_void_p, c_void_p, c_void_p]),
    "gfx_graph_destroy": (c_int, [c_void_p]),
    "gfx_graph_max_degree": (c_int64, [c_void_p]),
    "gfx_graph_trim": (c_int, [c_void_p]),
    "gfx_graph_refresh": (c_int, [c_void_p]),
    "gfx_bfs": (c_int, [c_void_p, c_int64, c_int, c_int, c_int, c_double, c_double, c_int,
                        c_int, c_void_p, c_void_p, POINTER(IterRec), c_int64, POINTER(Stats)]),
    "gfx_bfs_batch": (c_int, [c_void_p, POINTER(c_int64), c_int64, c_int, c_double, c_double,
                              c_int, c_void_p, c_void_p, POINTER(c_float)]),
    "gfx_estimate_mf_mu": (c_int, [c_int64, c_int64, c_int64, c_int64, c_int,
                                   POINTER(c_double), POINTER(c_double)]),
    "gfx_sssp": (c_int, [c_void_p, c_int64, c_double, c_void_p, c_void_p, POINTER(IterRec),
                         c_int64, POINTER(Stats)]),
    "gfx_bc": (c_int, [c_void_p, POINTER(c_int64), c_int64, c_void_p, POINTER(Stats)]),
    "gfx_cc": (c_int, [c_void_p, c_void_p, POINTER(c_int64), POINTER(Stats)]),
    "gfx_pagerank": (c_int, [c_void_p, c_double, c_double, c_int64, c_void_p, POINTER(Stats)]),
    "gfx_tc_orient": (c_int, [c_void_p, POINTER(c_int64)]),
    "gfx_tc_count": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int64),
                             POINTER(Stats)]),
    "gfx_segmented_intersect": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                        POINTER(c_int64)]),
    "gfx_advance": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, POINTER(FunctorArgs),
                            c_void_p, c_int64, POINTER(c_int64), POINTER(c_int64)]),
    "gfx_advance_fused": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, POINTER(FunctorArgs),
                                  c_int, POINTER(FunctorArgs), c_void_p, c_int64,
                                  POINTER(c_int64), POINTER(c_int64)]),
    "gfx_pull_advance": (c_int, [c_void_p, c_void_p, c_int64, c_int, POINTER(FunctorArgs),
                                 c_void_p, POINTER(c_int64), c_void_p, POINTER(c_int64),
                                 POINTER(c_int64)]),
    "gfx_vertex_mask": (c_int, [c_void_p, c_void_p, c_int64, c_int, POINTER(FunctorArgs),
                                c_void_p]),
    "gfx_scan_offsets": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p,
                                 POINTER(c_int64)]),
    "gfx_gather": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_int64,
                           c_void_p, c_void_p, c_void_p, c_void_p]),
    "gfx_graph_build_csc": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "gfx_select_i64": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p,
                               POINTER(c_int64)]),
    "gfx_mark_items": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "gfx_bitmap_test_and_set": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "gfx_unvisited": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_void_p,
                              POINTER(c_int64)]),
    "gfx_cull_stage": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int64, c_int64, c_int64,
                               c_void_p]),
    "gfx_atomic_min": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                               c_void_p]),
    "gfx_atomic_add": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_double,
                               c_int64]),
    "gfx_compare_and_swap": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int64, c_int64,
                                     c_void_p, c_int64, c_void_p, c_void_p]),
    "gfx_filter": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, POINTER(FunctorArgs),
                           c_int64, c_void_p, POINTER(c_int64)]),
    "gfx_compute": (c_int, [c_void_p, c_void_p, c_int64, c_int, POINTER(FunctorArgs), c_void_p]),
    "gfx_segmented_intersect_list": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                             c_void_p]),
    "gfx_csr_pack_size": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_void_p,
                                  POINTER(c_int64)]),
    "gfx_csr_pack": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_void_p, c_void_p, c_void_p]),
    "gfx_csr_unpack": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int,
                               c_int]),
    "gfx_graph_rebuild_upper": (c_int, [c_void_p, c_void_p, c_void_p, c_int64]),
    "gfx_rmat_keys": (c_int, [c_void_p, c_int, c_int, POINTER(c_double), c_uint64, c_uint64,
                              c_uint64, c_uint64, c_int, c_void_p, POINTER(c_int64)]),
    "gfx_keys_to_csr": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "gfx_assign_weights": (c_int, [c_void_p, c_int64, c_int64, c_uint64, c_uint64, c_uint64,
                                   c_uint64, c_void_p]),
    "gfx_dist_partition_sizes": (c_int, [c_void_p, c_int, c_int, POINTER(c_int64),
                                         POINTER(c_int64)]),
    "gfx_dist_partition": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "gfx_dbfs_create": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p, c_void_p,
                                c_int64, c_int64, POINTER(c_void_p)]),
    "gfx_dbfs_destroy": (c_int, [c_void_p]),
    "gfx_dbfs_words": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64)]),
    "gfx_dbfs_bind": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                              c_void_p, c_void_p, c_void_p, c_void_p]),
    "gfx_dbfs_reset": (c_int, [c_void_p, c_int64, POINTER(c_int64)]),
    "gfx_dbfs_push_expand": (c_int, [c_void_p, c_int32]),
    "gfx_dbfs_push_claim": (c_int, [c_void_p, c_int64, c_int32]),
    "gfx_dbfs_pull_prepare": (c_int, [c_void_p]),
    "gfx_dbfs_pull": (c_int, [c_void_p, c_int32]),
    "gfx_dbfs_commit": (c_int, [c_void_p, c_int64]),
    "gfx_dist_partition_weights": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "gfx_dsssp_create": (c_int, [c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                 c_int64, c_int64, POINTER(c_void_p)]),
    "gfx_dsssp_destroy": (c_int, [c_void_p]),
    "gfx_dsssp_bind": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                               c_void_p]),
    "gfx_dsssp_reset": (c_int, [c_void_p, c_int64, POINTER(c_int64)]),
    "gfx_dsssp_relax": (c_int, [c_void_p]),
    "gfx_dsssp_apply": (c_int, [c_void_p, c_int64]),
    "gfx_dsssp_split": (c_int, [c_void_p, c_double]),
    "gfx_dsssp_refar": (c_int, [c_void_p, c_double, c_int, c_int64]),
    "gfx_dsssp_result": (c_int, [c_void_p, c_void_p, c_void_p]),
    "gfx_nccl_load": (c_int, [c_char_p]),
    "gfx_nccl_unique_id": (c_int, [c_void_p]),
    "gfx_nccl_comm_create": (c_int, [c_void_p, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "gfx_nccl_comm_destroy": (c_int, [c_void_p]),
    "gfx_dbfs_run": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_double, c_double, c_int,
                             POINTER(IterRec), c_int64, POINTER(Stats)]),
    "gfx_dbfs_run_comm": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_double, c_double, c_int,
                                  POINTER(IterRec), c_int64, POINTER(Stats)]),
    "gfx_pdbfs_create_virtual": (c_int, [c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p,
                                         c_void_p, c_void_p, POINTER(c_void_p)]),
    "gfx_pdbfs_destroy": (c_int, [c_void_p]),
    "gfx_pdbfs_create_rank": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p,
                                      c_void_p, c_int64, c_int64, POINTER(c_void_p)]),
    "gfx_pdbfs_local_nnz": (c_int, [c_void_p, POINTER(c_int64)]),
    "gfx_pdbfs_export": (c_int, [c_void_p, c_void_p]),
    "gfx_pdbfs_import": (c_int, [c_void_p, c_void_p, c_int64]),
    "gfx_pdbfs_run": (c_int, [c_void_p, c_int64, c_int, c_double, c_double, c_int, c_void_p,
                              c_void_p, POINTER(IterRec), c_int64, POINTER(Stats)]),
    "gfx_pdbfs_batch": (c_int, [c_void_p, c_int64, c_int64, c_int, c_double, c_double, c_int,
                                POINTER(c_float)]),
    "gfx_pdsssp_create_virtual": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p, POINTER(c_void_p)]),
    "gfx_pdsssp_create_rank": (c_int, [c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p,
                                       c_void_p, c_int64, c_int64, POINTER(c_void_p)]),
    "gfx_pdsssp_export": (c_int, [c_void_p, c_void_p]),
    "gfx_pdsssp_import": (c_int, [c_void_p, c_void_p]),
    "gfx_pdsssp_destroy": (c_int, [c_void_p]),
    "gfx_pdsssp_run": (c_int, [c_void_p, c_int64, c_double, c_void_p, c_void_p, POINTER(IterRec),
                               c_int64, POINTER(Stats)]),
    "gfx_pdsssp_batch": (c_int, [c_void_p, c_int64, c_int64, c_double, POINTER(c_float)]),
    "gfx_debug_gridsync": (c_int, [c_void_p, c_int, c_int, c_int, c_int, POINTER(c_float)]),
    "gfx_debug_atomics": (c_int, [c_void_p, c_int, c_int, c_int, POINTER(c_double)]),
    "gfx_debug_chase": (c_int, [c_void_p, c_void_p, c_int, ctypes.c_uint32, POINTER(c_double)]),
    "gfx_debug_expand": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_int32,
                                 POINTER(c_float), POINTER(c_int64)]),
}

_lib = None
_lib_lock = threading.Lock()


class NativeError(RuntimeError):
    pass


def load_library() -> ctypes.CDLL:
    """Load libgfx.so (fails loudly when it has not been built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = LIB_PATH
        override = os.environ.get("GFX_LIB_PATH")  # A/B experiments against another build
        if override:
            path = Path(override)
        if not path.exists():
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_1701_01170_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            if override and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(status: int, what: str = "") -> None:
    if status == GFX_OK:
        return
    msg = load_library().gfx_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == GFX_EINVAL:
        raise ValueError(msg)
    if status == GFX_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load_library(), name)(*args), name)


class Context:
    """One libgfx context per CUDA device, ordered on torch's current stream."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1701_01170_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        lib = load_library()
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream(device).cuda_stream
        h = c_void_p()
        check(lib.gfx_ctx_create(device, c_void_p(stream), ctypes.byref(h)), "gfx_ctx_create")
        self.handle = h
        self.sm_count = lib.gfx_ctx_sm_count(h)

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        import torch

        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls(device)
            cls._by_device[device] = ctx
        return ctx

    def sync(self) -> None:
        call("gfx_ctx_sync", self.handle)

    def set_stats(self, detail: int) -> None:
        call("gfx_ctx_set_stats", self.handle, int(detail))

    def set_timing(self, enabled: bool) -> None:
        call("gfx_ctx_set_timing", self.handle, int(bool(enabled)))


def launch_count() -> int:
    return int(load_library().gfx_launch_count())


def ptr(t) -> c_void_p:
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return c_void_p(0)
    return c_void_p(t.data_ptr())


def estimate_mf_mu(n: int, m: int, n_f: int, n_u: int, mu_edge_based: bool = False):
    """Host C replica of the direction estimate (pure host code, no GPU)."""
    mf, mu = c_double(), c_double()
    call("gfx_estimate_mf_mu", n, m, n_f, n_u, int(mu_edge_based), ctypes.byref(mf),
         ctypes.byref(mu))
    return mf.value, mu.value


def env_flag(name: str, default: str = "0") -> bool:
    return os.environ.get(name, default) not in ("", "0", "false", "False")
