"""paper_2108_04167_b200 — B200 (sm_100a) hot path of ADMM + HSS kernel SVMs (arXiv 2108.04167).

Thin Python layer over the C-ABI library libsvmhss.so (include/svmhss.h): the same
entry-point names, argument marshalling only.  PyTorch is used for device memory and
streams; every computational step runs in the library's CUDA kernels.  Importing this
package loads the library and raises if it is missing (no CPU fallback).

    H = hss_build(F, h=..., leaf_size=..., rel_tol=..., max_rank=..., ...)
    U = hss_ulv_factor(H, beta)
    out = admm_svm_train(U, y, C=[...], max_it=...)
    dv, labels = svm_predict(F, y, out["z"], h, out["bias"], Ftest)
"""
from __future__ import annotations

import contextlib
import ctypes as ct

import numpy as np

from . import _lib
from ._lib import ALLGATHER_FN, AdmmOpts, AdmmStats, HssError, HssOpts, HssStats, UlvStats, check, ptr

_L = _lib.load()

__all__ = ["Comm", "hss_build", "hss_ulv_factor", "admm_svm_train", "svm_predict", "svm_train_predict_host",
           "hss_pool_trim",
           "hss_omega", "hss_tree", "hss_kernel_matmul", "hss_kernel_block", "HSS", "ULV", "HssError",
           "version"]


def version() -> str:
    return _L.hss_version().decode()


def launch_count() -> int:
    """Kernels launched by libsvmhss in this process (CUDA-graph replays included)."""
    return int(_L.hss_launch_count())


def _host_allgather(group):
    """hss_allgather_fn over torch.distributed (any backend that takes CPU tensors, e.g. gloo):
    argument marshalling only — the bytes are the library's, gathered rank-major."""
    import torch
    import torch.distributed as dist

    def cb(ctx, send, recv, nbytes):
        try:
            world = dist.get_world_size(group)
            if nbytes == 0:
                return 0
            sv = np.ctypeslib.as_array((ct.c_uint8 * nbytes).from_address(send))
            rv = np.ctypeslib.as_array((ct.c_uint8 * (nbytes * world)).from_address(recv))
            st, rt = torch.from_numpy(sv), torch.from_numpy(rv)
            dist.all_gather(list(rt.chunk(world)), st, group=group)
            return 0
        except Exception as e:  # noqa: BLE001 - reported to the library as a failed exchange
            print(f"[svmhss] host allgather failed: {e!r}")
            return 1

    return ALLGATHER_FN(cb)


class Comm:
    """Subtree-sharding communicator (hss_comm_t).

    Comm.nccl(): the library's own NCCL communicator (device buffers, graph-capturable); the
    128-byte unique id is created by rank 0 and broadcast over torch.distributed.
    Comm.host(): exchanges through a torch.distributed host group (e.g. gloo) — P ranks may then
    share fewer GPUs (tests)."""

    def __init__(self, handle, rank, world, keep=None):
        self._h, self.rank, self.world, self._keep = handle, rank, world, keep

    @classmethod
    def nccl(cls, group=None):
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            check(_L.hss_comm_nccl_id(uid.ctypes.data))
        t = torch.from_numpy(uid)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        uid = np.ascontiguousarray(t.cpu().numpy())
        hdl = ct.c_void_p()
        check(_L.hss_comm_init_nccl(world, rank, uid.ctypes.data, ct.byref(hdl)))
        return cls(hdl.value, rank, world)

    @classmethod
    def host(cls, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        fn = _host_allgather(group)
        hdl = ct.c_void_p()
        check(_L.hss_comm_init_host(world, rank, fn, None, ct.byref(hdl)))
        return cls(hdl.value, rank, world, keep=fn)

    @property
    def handle(self):
        return self._h

    def info(self):
        """dict(nranks, rank, device_api): device_api = 1 when the per-iteration exchange runs
        in-kernel through the NCCL device API."""
        a, b, c = ct.c_int32(), ct.c_int32(), ct.c_int32()
        check(_L.hss_comm_info(self.handle, ct.byref(a), ct.byref(b), ct.byref(c)))
        return dict(nranks=a.value, rank=b.value, device_api=c.value)

    def exchange_test(self, send):
        """Debug: one exchange of `send` (CUDA float64, count values) through the per-iteration
        path; returns (nranks * count) values, rank-major."""
        import torch
        _cuda_f64(send, "send")
        recv = torch.empty(self.world * send.numel(), dtype=torch.float64, device=send.device)
        ctx, d = _on_device(send)
        with ctx:
            check(_L.hss_comm_exchange_test(self.handle, ptr(send), send.numel(), ptr(recv), _stream(None, d)))
        return recv

    def free(self):
        if self._h is not None:
            _L.hss_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _cuda_f64(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous")
    return t


def _shape(cond, msg):
    if not cond:
        raise ValueError(msg)


def _on_device(*tensors):
    """Every call runs with the tensors' device current (kernels, stream and the library's pool
    of that device); all tensor arguments must share it."""
    import torch
    devs = {t.device for t in tensors if isinstance(t, torch.Tensor)}
    _shape(len(devs) <= 1, f"tensor arguments on different devices: {sorted(map(str, devs))}")
    if not devs:
        return contextlib.nullcontext(), None
    d = devs.pop()
    return torch.cuda.device(d), d


def _stream(stream, device=None):
    return _lib.stream_handle(stream, device)


class HSS:
    """Handle of a compressed kernel K~ (hss_t)."""

    def __init__(self, handle, n, r, h, device=None):
        self._h = handle
        self.n, self.r, self.h = n, r, h
        self.device = device

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("HSS handle freed")
        return self._h

    def info(self):
        st = HssStats()
        check(_L.hss_info(self.handle, ct.byref(st), None, None, None))
        d = {f: getattr(st, f) for f, _ in HssStats._fields_}
        nn = 2 ** (st.L + 1) - 1
        perm = np.empty(self.n, dtype=np.int64)
        ranks = np.empty(nn, dtype=np.int32)
        check(_L.hss_info(self.handle, None, perm.ctypes.data, ranks.ctypes.data, None))
        ksum = int(ranks[ranks > 0].sum())
        skel = np.empty(max(1, ksum), dtype=np.int64)
        check(_L.hss_info(self.handle, None, None, None, skel.ctypes.data))
        d.update(perm=perm, ranks=ranks, skeletons=skel[:ksum])
        return d

    def node(self, t):
        rows, k = ct.c_int32(), ct.c_int32()
        check(_L.hss_node(self.handle, t, ct.byref(rows), ct.byref(k), None, None, None))
        return rows.value, k.value

    def node_generators(self, t, L, k_children=None):
        rows, k = self.node(t)
        U = np.zeros((rows, max(k, 0)))
        D = None
        B = None
        lvl = int(np.floor(np.log2(t + 1)))
        if lvl == L:
            D = np.zeros((rows, rows))
        if lvl < L:
            ka = self.node(2 * t + 1)[1]
            kb = self.node(2 * t + 2)[1]
            B = np.zeros((ka, kb))
        check(_L.hss_node(self.handle, t, None, None, U.ctypes.data if k > 0 else None,
                          B.ctypes.data if B is not None and B.size else None,
                          D.ctypes.data if D is not None else None))
        return dict(rows=rows, k=k, U=U if k >= 0 else None, B=B, D=D)

    def matvec(self, v, stream=None):
        import torch
        _cuda_f64(v, "v")
        _shape(v.dim() in (1, 2) and v.shape[0] == self.n, f"v must have {self.n} rows (got {tuple(v.shape)})")
        _shape(self.device is None or v.device == self.device, "v is not on the HSS handle's device")
        nrhs = 1 if v.dim() == 1 else v.shape[1]
        out = torch.empty_like(v)
        ctx, d = _on_device(v)
        with ctx:
            check(_L.hss_matvec(self.handle, ptr(v), ptr(out), nrhs, _stream(stream, d)))
        return out

    def free(self):
        if self._h is not None:
            _L.hss_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class ULV:
    """Handle of the ULV factorization of K~ + beta I (ulv_t)."""

    def __init__(self, handle, hss, beta):
        self._h = handle
        self.hss, self.beta = hss, beta

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("ULV handle freed")
        return self._h

    def info(self):
        st = UlvStats()
        check(_L.ulv_info(self.handle, ct.byref(st)))
        return {f: getattr(st, f) for f, _ in UlvStats._fields_}

    def solve(self, b, stream=None):
        import torch
        _cuda_f64(b, "b")
        n = self.hss.n
        _shape(b.dim() in (1, 2) and b.shape[0] == n, f"b must have {n} rows (got {tuple(b.shape)})")
        _shape(self.hss.device is None or b.device == self.hss.device, "b is not on the ULV handle's device")
        nrhs = 1 if b.dim() == 1 else b.shape[1]
        x = torch.empty_like(b)
        ctx, d = _on_device(b)
        with ctx:
            check(_L.ulv_solve(self.handle, ptr(b), ptr(x), nrhs, _stream(stream, d)))
        return x

    def free(self):
        if self._h is not None:
            _L.ulv_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


SAMPLING = {"sketch": 0, "ann": 1}
INTERP = {"id": 0, "spd": 1}


def make_opts(leaf_size, rel_tol=0.0, abs_tol=0.0, max_rank=64, oversample=16, omega_seed=0,
              tree_seed=0, ranks=None, comm=None, sampling="sketch", ann_neighbors=64, ann_trees=4,
              ann_leaf=256, ann_seed=0, adaptive_s0=0, adaptive_ds=0, perm=None, skeletons=None,
              interp="id", spd_eps=1e-12):
    if interp not in INTERP:
        raise ValueError(f"interp must be one of {sorted(INTERP)}, got {interp!r}")
    if sampling not in SAMPLING:
        raise ValueError(f"sampling must be one of {sorted(SAMPLING)}, got {sampling!r}")
    o = HssOpts()
    o.interp, o.spd_eps = INTERP[interp], float(spd_eps)
    o.adaptive_s0, o.adaptive_ds = int(adaptive_s0), int(adaptive_ds)
    o.comm = comm.handle if comm is not None else None
    o.sampling = SAMPLING[sampling]
    o.ann_neighbors, o.ann_trees, o.ann_leaf, o.ann_seed = int(ann_neighbors), int(ann_trees), int(ann_leaf), int(ann_seed)
    o.leaf_size, o.rel_tol, o.abs_tol = int(leaf_size), float(rel_tol), float(abs_tol)
    o.max_rank, o.oversample = int(max_rank), int(oversample)
    o.omega_seed, o.tree_seed = int(omega_seed), int(tree_seed)
    keep = []
    if ranks is not None:
        kr = np.ascontiguousarray(np.asarray(ranks, dtype=np.int32))
        o.ranks = kr.ctypes.data_as(ct.POINTER(ct.c_int32))
        keep.append(kr)
    if perm is not None:
        kp = np.ascontiguousarray(np.asarray(perm, dtype=np.int64))
        o.perm = kp.ctypes.data_as(ct.POINTER(ct.c_int64))
        keep.append(kp)
    if skeletons is not None:
        ks = np.ascontiguousarray(np.asarray(skeletons, dtype=np.int64))
        o.skeletons = ks.ctypes.data_as(ct.POINTER(ct.c_int64))
        keep.append(ks)
    return o, keep


def hss_build(F, h, leaf_size, rel_tol=0.0, abs_tol=0.0, max_rank=64, oversample=16, omega_seed=0,
              tree_seed=0, ranks=None, comm=None, sampling="sketch", ann_neighbors=64, ann_trees=4,
              ann_leaf=256, ann_seed=0, adaptive_s0=0, adaptive_ds=0, perm=None, skeletons=None,
              interp="id", spd_eps=1e-12, stream=None) -> HSS:
    """hss_build (Alg. 3 line 1): F is a CUDA float64 (n, r) tensor, original order
    (all n points on every rank when `comm` shards the tree).  sampling="ann" selects HSS-ANN
    column sampling instead of the randomized sketch.  perm / skeletons (host
    arrays) import a tree / fixed skeletons (parity modes; include/svmhss.h).  interp="spd"
    selects the SPD-preserving kernel interpolation onto the skeletons (N4; include/svmhss.h)."""
    _cuda_f64(F, "F")
    _shape(F.dim() == 2, "F must be (n, r)")
    n, r = F.shape
    if perm is not None:
        _shape(np.asarray(perm).shape == (n,), f"perm must have {n} entries")
    o, keep = make_opts(leaf_size, rel_tol, abs_tol, max_rank, oversample, omega_seed, tree_seed, ranks, comm,
                        sampling, ann_neighbors, ann_trees, ann_leaf, ann_seed, adaptive_s0, adaptive_ds,
                        perm, skeletons, interp, spd_eps)
    hdl = ct.c_void_p()
    ctx, d = _on_device(F)
    with ctx:
        check(_L.hss_build(ptr(F), n, r, float(h), ct.byref(o), _stream(stream, d), ct.byref(hdl)))
    del keep
    H = HSS(hdl.value, n, r, h, F.device)
    H.comm = comm  # keep the Python object alive with the handle
    return H


def hss_ulv_factor(H: HSS, beta, stream=None) -> ULV:
    """hss_ulv_factor."""
    import torch
    hdl = ct.c_void_p()
    ctx = torch.cuda.device(H.device) if H.device is not None else contextlib.nullcontext()
    with ctx:
        check(_L.hss_ulv_factor(H.handle, float(beta), _stream(stream, H.device), ct.byref(hdl)))
    return ULV(hdl.value, H, beta)


def admm_svm_train(U: ULV, y, C, max_it, trace_every=0, margin_eps_rel=0.0, want_mu=True,
                   stream=None):
    """admm_svm_train (Alg. 2 / Alg. 3).  y: CUDA float64 (n,), +-1.
    Returns dict(z (n, nC), mu, bias[nC], obj[nC], stats, trace_z, trace_mu)."""
    import torch
    _cuda_f64(y, "y")
    n = U.hss.n
    _shape(y.dim() == 1 and y.shape[0] == n, f"y must have shape ({n},) (got {tuple(y.shape)})")
    _shape(U.hss.device is None or y.device == U.hss.device, "y is not on the ULV handle's device")
    Cs = np.ascontiguousarray(np.atleast_1d(np.asarray(C, dtype=np.float64)))
    nC = Cs.shape[0]
    z = torch.empty((n, nC), dtype=torch.float64, device=y.device)
    mu = torch.empty_like(z) if want_mu else None
    bias = np.zeros(nC)
    obj = np.zeros(nC)
    opts = AdmmOpts()
    opts.margin_eps_rel = float(margin_eps_rel)
    tz = tm = None
    if trace_every:
        nt = -(-int(max_it) // int(trace_every))
        tz = torch.empty((nt, n, nC), dtype=torch.float64, device=y.device)
        tm = torch.empty_like(tz)
        opts.trace_every, opts.trace_z, opts.trace_mu = int(trace_every), ptr(tz), ptr(tm)
    st = AdmmStats()
    ctx, d = _on_device(y)
    with ctx:
        check(_L.admm_svm_train(U.handle, ptr(y), Cs.ctypes.data, nC, int(max_it), ct.byref(opts), ptr(z),
                                ptr(mu), bias.ctypes.data, obj.ctypes.data, ct.byref(st), _stream(stream, d)))
    return dict(z=z, mu=mu, bias=bias, obj=obj, trace_z=tz, trace_mu=tm,
                stats={f: getattr(st, f) for f, _ in AdmmStats._fields_})


def svm_predict(Ftrain, y, z, h, bias, Ftest, comm=None, stream=None):
    """svm_predict: dv = K(Ftest, Ftrain) (y o z) + bias; labels = sign (0 -> +1).
    y: (n,) labels, z: (n,) or (n, nC) dual variables (admm_svm_train's z), bias: nC values.
    comm: shard the test points over its ranks (every rank gets the full outputs)."""
    import torch
    for t, nm in ((Ftrain, "Ftrain"), (y, "y"), (z, "z"), (Ftest, "Ftest")):
        _cuda_f64(t, nm)
    _shape(Ftrain.dim() == 2 and Ftest.dim() == 2, "Ftrain and Ftest must be 2-D")
    n, r = Ftrain.shape
    m = Ftest.shape[0]
    _shape(Ftest.shape[1] == r, f"Ftest must have {r} columns (got {Ftest.shape[1]})")
    _shape(y.dim() == 1 and y.shape[0] == n, f"y must have shape ({n},)")
    _shape(z.dim() in (1, 2) and z.shape[0] == n, f"z must have {n} rows")
    nC = 1 if z.dim() == 1 else z.shape[1]
    b = np.ascontiguousarray(np.atleast_1d(np.asarray(bias, dtype=np.float64)))
    _shape(b.shape == (nC,), f"bias must have {nC} entries (got {b.shape[0]})")
    dv = torch.empty((m, nC), dtype=torch.float64, device=Ftrain.device)
    lab = torch.empty((m, nC), dtype=torch.int8, device=Ftrain.device)
    ctx, d = _on_device(Ftrain, y, z, Ftest)
    with ctx:
        check(_L.svm_predict(ptr(Ftrain), ptr(y), ptr(z), n, r, float(h), b.ctypes.data, nC, ptr(Ftest), m,
                             ptr(dv), ptr(lab), comm.handle if comm is not None else None, _stream(stream, d)))
    return dv, lab


def hss_pool_trim():
    """Release the memory the library keeps reserved in its pool on the current device."""
    check(_L.hss_pool_trim())


def svm_train_predict_host(F, y, h, beta, C, max_it, Ftest=None, **opt_kw):
    """End-to-end on HOST numpy buffers (Alg. 3): copies in, build, factor, ADMM, bias,
    predict, copies out.  Returns dict(z, bias, obj, labels, timings_ms)."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, r = F.shape
    _shape(y.shape == (n,), f"y must have shape ({n},)")
    Cs = np.ascontiguousarray(np.atleast_1d(np.asarray(C, dtype=np.float64)))
    nC = Cs.shape[0]
    if Ftest is not None:
        _shape(np.asarray(Ftest).ndim == 2 and np.asarray(Ftest).shape[1] == r, f"Ftest must have {r} columns")
    o, keep = make_opts(**opt_kw)
    z = np.zeros((n, nC))
    bias, obj = np.zeros(nC), np.zeros(nC)
    tim = np.zeros(8)
    if Ftest is not None:
        Ft = np.ascontiguousarray(Ftest, dtype=np.float64)
        m = Ft.shape[0]
        lab = np.zeros((m, nC), dtype=np.int8)
    else:
        Ft, m, lab = None, 0, None
    check(_L.svm_train_predict_host(F.ctypes.data, y.ctypes.data, n, r, float(h), ct.byref(o),
                                    float(beta), Cs.ctypes.data, nC, int(max_it),
                                    Ft.ctypes.data if Ft is not None else None, m, z.ctypes.data,
                                    bias.ctypes.data, obj.ctypes.data,
                                    lab.ctypes.data if lab is not None else None, tim.ctypes.data))
    del keep
    names = ["h2d", "build", "factor", "admm", "bias", "predict", "d2h", "total"]
    return dict(z=z, bias=bias, obj=obj, labels=lab, timings_ms=dict(zip(names, tim.tolist())))


# ---- debug / parity exports
def hss_ann_lists(F, kappa, trees, leaf, seed, stream=None):
    """N1 ANN lists of the rows of F (original order): (idx (n, kappa) int64, d (n, kappa))."""
    import torch
    _cuda_f64(F, "F")
    n, r = F.shape
    idx = torch.empty((n, kappa), dtype=torch.int64, device=F.device)
    d = torch.empty((n, kappa), dtype=torch.float64, device=F.device)
    check(_L.hss_ann_lists(ptr(F), n, r, int(kappa), int(trees), int(leaf), int(seed), ptr(idx), ptr(d),
                           _stream(stream)))
    return idx, d


def hss_omega(seed, idx, s, stream=None):
    import torch
    idx = idx.to(torch.int64).contiguous()
    out = torch.empty((idx.shape[0], s), dtype=torch.float64, device=idx.device)
    check(_L.hss_omega(int(seed), ptr(idx), idx.shape[0], int(s), ptr(out), _stream(stream)))
    return out


def hss_tree(F, leaf_size, tree_seed, stream=None):
    import torch
    _cuda_f64(F, "F")
    perm = torch.empty(F.shape[0], dtype=torch.int64, device=F.device)
    check(_L.hss_tree(ptr(F), F.shape[0], F.shape[1], int(leaf_size), int(tree_seed), ptr(perm),
                      _stream(stream)))
    return perm


def hss_kernel_matmul(Fa, Fb, h, W, same_set=False, stream=None):
    import torch
    for t, nm in ((Fa, "Fa"), (Fb, "Fb"), (W, "W")):
        _cuda_f64(t, nm)
    S = torch.empty((Fa.shape[0], W.shape[1]), dtype=torch.float64, device=Fa.device)
    _shape(Fb.shape[1] == Fa.shape[1] and W.shape[0] == Fb.shape[0], "hss_kernel_matmul: shape mismatch")
    ctx, d = _on_device(Fa, Fb, W)
    with ctx:
        check(_L.hss_kernel_matmul(ptr(Fa), Fa.shape[0], ptr(Fb), Fb.shape[0], Fa.shape[1], float(h), ptr(W),
                                   W.shape[1], int(bool(same_set)), ptr(S), _stream(stream, d)))
    return S


def hss_kernel_block(Fa, Fb, h, stream=None):
    import torch
    _cuda_f64(Fa, "Fa")
    _cuda_f64(Fb, "Fb")
    K = torch.empty((Fa.shape[0], Fb.shape[0]), dtype=torch.float64, device=Fa.device)
    check(_L.hss_kernel_block(ptr(Fa), Fa.shape[0], ptr(Fb), Fb.shape[0], Fa.shape[1], float(h), ptr(K),
                              _stream(stream)))
    return K
