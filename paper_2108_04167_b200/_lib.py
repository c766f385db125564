"""ctypes binding of libsvmhss.so (include/svmhss.h) — argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only converts torch
device tensors / numpy arrays to pointers and sizes.  There is NO fallback: if the
library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsvmhss.so")

HSS_ERRORS = {0: "HSS_OK", -1: "HSS_EINVAL", -2: "HSS_ENOMEM", -3: "HSS_ECUDA", -4: "HSS_ENCCL",
              -5: "HSS_ENOTSPD", -6: "HSS_EW1"}


class HssError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{HSS_ERRORS.get(code, code)}: {msg}")
        self.code = code


class HssOpts(ct.Structure):
    _fields_ = [("leaf_size", ct.c_int32), ("rel_tol", ct.c_double), ("abs_tol", ct.c_double),
                ("max_rank", ct.c_int32), ("oversample", ct.c_int32), ("omega_seed", ct.c_uint64),
                ("tree_seed", ct.c_uint64), ("ranks", ct.POINTER(ct.c_int32)), ("comm", ct.c_void_p),
                ("sampling", ct.c_int32), ("ann_neighbors", ct.c_int32), ("ann_trees", ct.c_int32),
                ("ann_leaf", ct.c_int32), ("ann_seed", ct.c_uint64),
                ("adaptive_s0", ct.c_int32), ("adaptive_ds", ct.c_int32),
                ("perm", ct.POINTER(ct.c_int64)), ("skeletons", ct.POINTER(ct.c_int64)),
                ("interp", ct.c_int32), ("spd_eps", ct.c_double)]


# int (*hss_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes)
ALLGATHER_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_size_t)


class HssStats(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("r", ct.c_int32), ("L", ct.c_int32), ("s", ct.c_int32),
                ("leaf_size", ct.c_int32), ("max_rank_used", ct.c_int32), ("cap_hits", ct.c_int32),
                ("passthrough", ct.c_int32), ("generator_bytes", ct.c_int64),
                ("ms_tree", ct.c_double), ("ms_omega", ct.c_double), ("ms_sketch", ct.c_double),
                ("ms_compress", ct.c_double), ("s_used", ct.c_int32), ("sample_rounds", ct.c_int32)]


class UlvStats(ct.Structure):
    _fields_ = [("beta", ct.c_double), ("factor_bytes", ct.c_int64), ("ms_factor", ct.c_double),
                ("factor_flops", ct.c_double)]


class AdmmOpts(ct.Structure):
    _fields_ = [("trace_every", ct.c_int32), ("trace_z", ct.c_void_p), ("trace_mu", ct.c_void_p),
                ("margin_eps_rel", ct.c_double)]


class AdmmStats(ct.Structure):
    _fields_ = [("w1", ct.c_double), ("ms_precompute", ct.c_double), ("ms_loop", ct.c_double),
                ("ms_bias", ct.c_double), ("iterations", ct.c_int32), ("graph", ct.c_int32),
                ("kernel_launches_per_iter", ct.c_int64)]


EXPORTS = ["hss_build", "hss_info", "hss_matvec", "hss_ulv_factor", "ulv_info", "ulv_solve",
           "admm_svm_train", "svm_predict", "svm_train_predict_host", "hss_omega", "hss_tree",
           "hss_kernel_matmul", "hss_kernel_block", "hss_node", "hss_free", "ulv_free",
           "hss_last_error", "hss_version", "hss_launch_count", "hss_comm_nccl_id",
           "hss_comm_init_nccl", "hss_comm_init_host", "hss_comm_free", "hss_ann_lists", "hss_pool_trim",
           "hss_comm_info", "hss_comm_exchange_test"]

_lib = None


def load():
    """Load the library (raises if absent — never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python paper_2108_04167_b200/build.py`")
    L = ct.CDLL(LIB_PATH)
    vp, i32, i64, u64, dbl = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_uint64, ct.c_double
    L.hss_build.argtypes = [vp, i64, i32, dbl, ct.POINTER(HssOpts), vp, ct.POINTER(vp)]
    L.hss_info.argtypes = [vp, ct.POINTER(HssStats), vp, vp, vp]
    L.hss_matvec.argtypes = [vp, vp, vp, i32, vp]
    L.hss_ulv_factor.argtypes = [vp, dbl, vp, ct.POINTER(vp)]
    L.ulv_info.argtypes = [vp, ct.POINTER(UlvStats)]
    L.ulv_solve.argtypes = [vp, vp, vp, i32, vp]
    L.admm_svm_train.argtypes = [vp, vp, vp, i32, i32, ct.POINTER(AdmmOpts), vp, vp, vp, vp,
                                 ct.POINTER(AdmmStats), vp]
    L.svm_predict.argtypes = [vp, vp, vp, i64, i32, dbl, vp, i32, vp, i64, vp, vp, vp, vp]
    L.hss_pool_trim.argtypes = []
    L.hss_comm_info.argtypes = [vp, ct.POINTER(i32), ct.POINTER(i32), ct.POINTER(i32)]
    L.hss_comm_exchange_test.argtypes = [vp, vp, i64, vp, vp]
    L.svm_train_predict_host.argtypes = [vp, vp, i64, i32, dbl, ct.POINTER(HssOpts), dbl, vp, i32,
                                         i32, vp, i64, vp, vp, vp, vp, vp]
    L.hss_omega.argtypes = [u64, vp, i64, i32, vp, vp]
    L.hss_ann_lists.argtypes = [vp, i64, i32, i32, i32, i32, u64, vp, vp, vp]
    L.hss_tree.argtypes = [vp, i64, i32, i32, u64, vp, vp]
    L.hss_kernel_matmul.argtypes = [vp, i64, vp, i64, i32, dbl, vp, i32, i32, vp, vp]
    L.hss_kernel_block.argtypes = [vp, i64, vp, i64, i32, dbl, vp, vp]
    L.hss_node.argtypes = [vp, i32, ct.POINTER(i32), ct.POINTER(i32), vp, vp, vp]
    L.hss_free.argtypes = [vp]
    L.hss_free.restype = None
    L.ulv_free.argtypes = [vp]
    L.ulv_free.restype = None
    L.hss_last_error.restype = ct.c_char_p
    L.hss_version.restype = ct.c_char_p
    L.hss_comm_nccl_id.argtypes = [vp]
    L.hss_comm_init_nccl.argtypes = [i32, i32, vp, ct.POINTER(vp)]
    L.hss_comm_init_host.argtypes = [i32, i32, ALLGATHER_FN, vp, ct.POINTER(vp)]
    L.hss_comm_free.argtypes = [vp]
    L.hss_comm_free.restype = None
    L.hss_launch_count.argtypes = []
    L.hss_launch_count.restype = ct.c_int64
    for name in EXPORTS:
        if name not in ("hss_free", "ulv_free", "hss_last_error", "hss_version", "hss_launch_count",
                        "hss_comm_free"):
            getattr(L, name).restype = ct.c_int
    _lib = L
    return L


def check(code: int):
    if code != 0:
        raise HssError(code, load().hss_last_error().decode())


def ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_handle(stream=None, device=None):
    """cudaStream_t of `stream`, else of the current stream of `device` (the tensors' device)."""
    import torch
    s = torch.cuda.current_stream(device) if stream is None else stream
    return s.cuda_stream
