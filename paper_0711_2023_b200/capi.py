"""Thin ctypes binding of libtucker.so (include/tucker.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  The module fails loudly (ImportError) when libtucker.so is missing;
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtucker.so")

TUCKER_INPUT_ON_DEVICE = 0x1
TUCKER_OUTPUT_ON_DEVICE = 0x2
TUCKER_HOST_COLLECTIVES = 0x4
# int fn(void* dev_buf, int64_t count, int dtype, void* stream, void* user)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p)
E_OOM = 8
E_CONVERGE = 10

# every symbol declared in include/tucker.h
EXPORTS = [
    "tucker_default_opts", "tucker_init", "hooi_sweep", "mp_sweep", "core_and_fit",
    "tucker_set_factors", "tucker_free", "tucker_strerror", "tucker_last_error",
    "tucker_debug_ttmc", "tucker_debug_gram", "tucker_debug_eig", "tucker_debug_smalldense",
    "tucker_debug_product", "tucker_debug_product_time", "tucker_csf_stats", "tucker_stats",
    "tucker_nccl_unique_id", "tucker_shard_bounds", "tucker_shard_info", "hooi_run", "mp_run",
    "tucker_hosvd", "sp_sweep", "sp_run", "tucker_set_factor", "tucker_set_allreduce",
    "tucker_time_ttmc", "tucker_csf_layout", "tucker_debug_gram_rows", "tucker_mp_overlap_times",
]


class tucker_opts(C.Structure):
    _fields_ = [
        ("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
        ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p),
        ("eig_oversample", C.c_int), ("eig_max_iter", C.c_int), ("eig_tol", C.c_double),
        ("flags", C.c_uint),
    ]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libtucker.so not built ({path}); run __graft_entry__.build()")
    lib = C.CDLL(path)
    P = C.c_void_p
    i64p = C.POINTER(C.c_int64)
    lib.tucker_default_opts.argtypes = [C.POINTER(tucker_opts)]
    lib.tucker_default_opts.restype = None
    lib.tucker_init.argtypes = [C.POINTER(P), C.c_int, i64p, i64p, C.c_int64, C.POINTER(P), P,
                                C.POINTER(P), C.POINTER(tucker_opts)]
    lib.hooi_sweep.argtypes = [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)]
    lib.mp_sweep.argtypes = [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)]
    lib.core_and_fit.argtypes = [P, P, C.POINTER(P), C.POINTER(C.c_double)]
    lib.tucker_set_factors.argtypes = [P, C.POINTER(P)]
    lib.tucker_free.argtypes = [P]
    lib.tucker_strerror.argtypes = [C.c_int]
    lib.tucker_strerror.restype = C.c_char_p
    lib.tucker_last_error.argtypes = [P]
    lib.tucker_last_error.restype = C.c_char_p
    lib.tucker_debug_ttmc.argtypes = [P, C.c_int, P]
    lib.tucker_debug_gram.argtypes = [P, C.c_int, C.c_int, P]
    lib.tucker_debug_eig.argtypes = [P, C.c_int, C.c_int, P, P, P]
    lib.tucker_stats.argtypes = [P, i64p, C.c_int]
    lib.tucker_debug_product.argtypes = [C.c_int, C.c_int, P, P, C.c_double, C.c_double, P, P]
    lib.tucker_debug_product_time.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.tucker_csf_stats.argtypes = [P, i64p]
    lib.tucker_csf_layout.argtypes = [P, i64p]
    lib.tucker_debug_gram_rows.argtypes = [P, C.c_int, C.c_int, C.c_int, i64p, P]
    lib.tucker_time_ttmc.argtypes = [P, C.c_int, C.c_int, C.POINTER(C.c_float)]
    lib.tucker_mp_overlap_times.argtypes = [P, C.POINTER(C.c_double), i64p, C.c_int]
    lib.tucker_nccl_unique_id.argtypes = [P]
    lib.tucker_hosvd.argtypes = [P, C.c_uint]
    lib.tucker_set_allreduce.argtypes = [P, P, P]
    lib.sp_sweep.argtypes = [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_float)]
    lib.sp_run.argtypes = [P, C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.tucker_set_factor.argtypes = [P, C.c_int, P, C.c_int]
    lib.hooi_run.argtypes = [P, C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.mp_run.argtypes = [P, C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.tucker_shard_bounds.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int, i64p]
    lib.tucker_shard_info.argtypes = [P, i64p]
    lib.tucker_debug_smalldense.argtypes = [C.c_int, C.c_int, P, P, P, P, C.c_int, C.c_double]
    for name in EXPORTS:
        if name not in ("tucker_default_opts", "tucker_strerror", "tucker_last_error"):
            getattr(lib, name).restype = C.c_int
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


class TuckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int, h=None, allow=()):
    if rc != 0 and rc not in allow:
        L = lib()
        detail = L.tucker_last_error(h).decode() if h else ""
        raise TuckerError(rc, L.tucker_strerror(rc).decode() + (": " + detail if detail else ""))
    return rc


def _ptr(a) -> int:
    """Address of a numpy array or a torch tensor (host or device)."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


# shapes of every live handle (dims, core), so calls that take factors can check them
_shapes: dict = {}


def _numel(a) -> int:
    return int(a.numel() if hasattr(a, "numel") else np.asarray(a).size)


def _check_array(a, what, dtype, shape=None, size=None, device=False):
    """The C side reads exactly the declared number of elements from these pointers:
    reject a wrong dtype, size or shape here instead of reading out of bounds."""
    if hasattr(a, "data_ptr"):  # torch tensor
        import torch
        tdt = {np.int32: torch.int32, np.float32: torch.float32}[dtype]
        if a.dtype != tdt:
            raise TypeError(f"{what}: dtype {a.dtype}, expected {tdt}")
        if not a.is_contiguous():
            raise ValueError(f"{what}: tensor must be contiguous")
        if device != a.is_cuda:
            raise ValueError(f"{what}: expected a {'device' if device else 'host'} tensor")
        got = tuple(a.shape)
    else:
        if device:
            raise ValueError(f"{what}: on_device=True needs torch CUDA tensors")
        got = np.shape(a)
    if shape is not None and tuple(got) != tuple(shape):
        raise ValueError(f"{what}: shape {tuple(got)}, expected {tuple(shape)}")
    if size is not None and _numel(a) != size:
        raise ValueError(f"{what}: {_numel(a)} elements, expected {size}")


def _check_factors(dims, core, U, device, what="U"):
    if len(U) != len(dims):
        raise ValueError(f"{what}: {len(U)} factors for an order-{len(dims)} tensor")
    for n, u in enumerate(U):
        _check_array(u, f"{what}[{n}]", np.float32, shape=(dims[n], core[n]), device=device)


def tucker_init(dims, core, idx, vals, U0, *, device=0, stream=None, eig_oversample=0,
                eig_max_iter=0, eig_tol=0.0, on_device=False, output_on_device=False,
                rank=0, world=1, nccl_id=None, host_collectives=False):
    """Returns an opaque handle (int).  idx: list of N int32 arrays (0-based),
    vals: fp32, U0: list of N fp32 row-major I_n x J_n arrays.  Host numpy
    arrays, or torch CUDA tensors with on_device=True.  Multi-GPU: every rank
    passes the full tensor, its rank, the world size and the same 128-byte
    nccl_id (nccl_unique_id() on one rank, broadcast by the caller)."""
    L = lib()
    N = len(dims)
    dims = tuple(int(x) for x in dims)
    core = tuple(int(x) for x in core)
    if len(core) != N or len(idx) != N or len(U0) != N:
        raise ValueError(f"order {N}: need {N} core sizes, index arrays and factors "
                         f"(got {len(core)}, {len(idx)}, {len(U0)})")
    if not on_device:
        idx = [np.ascontiguousarray(a, dtype=np.int32) for a in idx]
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        U0 = [np.ascontiguousarray(u, dtype=np.float32) for u in U0]
    nnz = _numel(vals)
    _check_array(vals, "vals", np.float32, device=on_device)
    if not hasattr(vals, "data_ptr") and np.ndim(vals) != 1:
        raise ValueError("vals must be 1-D")
    for n, a in enumerate(idx):
        _check_array(a, f"idx[{n}]", np.int32, size=nnz, device=on_device)
        if np.ndim(a) != 1 and not hasattr(a, "data_ptr"):
            raise ValueError(f"idx[{n}] must be 1-D")
    _check_factors(dims, core, U0, on_device, "U0")
    o = tucker_opts()
    L.tucker_default_opts(C.byref(o))
    o.device = device
    o.stream = stream
    o.eig_oversample = eig_oversample
    o.eig_max_iter = eig_max_iter
    o.eig_tol = eig_tol
    o.flags = (TUCKER_INPUT_ON_DEVICE if on_device else 0) | (
        TUCKER_OUTPUT_ON_DEVICE if output_on_device else 0)
    o.rank = rank
    o.world = world
    if host_collectives:
        o.flags |= TUCKER_HOST_COLLECTIVES
    idbuf = None
    if nccl_id is not None:
        _load_torch_nccl()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        o.nccl_unique_id = C.cast(idbuf, C.c_void_p)
    d = (C.c_int64 * N)(*[int(x) for x in dims])
    j = (C.c_int64 * N)(*[int(x) for x in core])
    ip = (C.c_void_p * N)(*[_ptr(a) for a in idx])
    up = (C.c_void_p * N)(*[_ptr(u) for u in U0])
    h = C.c_void_p()
    rc = L.tucker_init(C.byref(h), N, d, j, nnz, ip, C.c_void_p(_ptr(vals)), up, C.byref(o))
    _check(rc)
    _shapes[h.value] = (dims, core, bool(on_device))
    return h.value


def hooi_sweep(h, sweeps, want_stage=False):
    fits = np.zeros(sweeps, dtype=np.float64)
    stage = np.zeros(sweeps * 4, dtype=np.float32)
    rc = lib().hooi_sweep(h, sweeps, fits.ctypes.data_as(C.POINTER(C.c_double)),
                          stage.ctypes.data_as(C.POINTER(C.c_float)) if want_stage else None)
    _check(rc, h, allow=(E_CONVERGE,))
    return (fits, stage.reshape(sweeps, 4), rc) if want_stage else fits


def mp_sweep(h, sweeps, want_fit=True, want_stage=False):
    fits = np.zeros(sweeps, dtype=np.float64)
    stage = np.zeros(sweeps * 4, dtype=np.float32)
    rc = lib().mp_sweep(h, sweeps, fits.ctypes.data_as(C.POINTER(C.c_double)) if want_fit else None,
                        stage.ctypes.data_as(C.POINTER(C.c_float)) if want_stage else None)
    _check(rc, h, allow=(E_CONVERGE,))
    return (fits, stage.reshape(sweeps, 4), rc) if want_stage else fits


def core_and_fit_into(h, core_out, U_out):
    """core_and_fit writing into caller buffers (numpy or torch, host or device
    according to the handle's output flag); returns the fit."""
    N = len(U_out) if U_out is not None else 0
    if h in _shapes:  # the library writes prod J and I_n x J_n elements into these
        dims, core, _ = _shapes[h]
        if core_out is not None and _numel(core_out) != int(np.prod(core)):
            raise ValueError(f"core_out: {_numel(core_out)} elements, expected {int(np.prod(core))}")
        if U_out is not None:
            if N != len(dims):
                raise ValueError(f"U_out: {N} buffers for an order-{len(dims)} tensor")
            for n, u in enumerate(U_out):
                if u is not None and _numel(u) != dims[n] * core[n]:
                    raise ValueError(f"U_out[{n}]: {_numel(u)} elements, expected {dims[n] * core[n]}")
    up = (C.c_void_p * N)(*[_ptr(u) if u is not None else None for u in U_out]) if U_out is not None else None
    fit = C.c_double()
    rc = lib().core_and_fit(h, C.c_void_p(_ptr(core_out)) if core_out is not None else None, up,
                            C.byref(fit))
    _check(rc, h)
    return fit.value


def core_and_fit(h, dims, core, want_core=True, want_factors=True):
    N = len(dims)
    G = np.zeros(int(np.prod(core)), dtype=np.float32) if want_core else None
    Us = [np.zeros((dims[n], core[n]), dtype=np.float32) for n in range(N)] if want_factors else None
    up = (C.c_void_p * N)(*[u.ctypes.data for u in Us]) if want_factors else None
    fit = C.c_double()
    rc = lib().core_and_fit(h, C.c_void_p(G.ctypes.data) if want_core else None, up, C.byref(fit))
    _check(rc, h)
    if want_core:
        G = G.reshape(tuple(core), order="F")  # mode-1 fastest
    return G, Us, fit.value


def tucker_set_factors(h, U):
    if not all(hasattr(u, "data_ptr") for u in U):
        U = [np.ascontiguousarray(u, dtype=np.float32) for u in U]
    if h in _shapes:
        dims, core, dev = _shapes[h]
        _check_factors(dims, core, U, dev)
    up = (C.c_void_p * len(U))(*[_ptr(u) for u in U])
    _check(lib().tucker_set_factors(h, up), h)


def tucker_free(h):
    if h:
        _shapes.pop(h, None)
        lib().tucker_free(h)


def tucker_debug_ttmc(h, mode, I, P):
    Y = np.zeros((I, P), dtype=np.float32)
    _check(lib().tucker_debug_ttmc(h, mode, C.c_void_p(Y.ctypes.data)), h)
    return Y


def tucker_debug_gram(h, algo, mode, I):
    S = np.zeros((I, I), dtype=np.float64)
    _check(lib().tucker_debug_gram(h, algo, mode, C.c_void_p(S.ctypes.data)), h)
    return S


def tucker_debug_gram_rows(h, algo, mode, rows, I):
    """Rows of the fp64 Gram (algo 0 HOOI, 1 MP) the next update of `mode` would use."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((rows.size, I), dtype=np.float64)
    _check(lib().tucker_debug_gram_rows(h, algo, mode, int(rows.size), rows.ctypes.data_as(C.POINTER(C.c_int64)),
                                        C.c_void_p(out.ctypes.data)), h)
    return out


def tucker_debug_eig(h, S, J):
    S = np.ascontiguousarray(S, dtype=np.float64)
    d = S.shape[0]
    U = np.zeros((d, J), dtype=np.float32)
    w = np.zeros(J, dtype=np.float64)
    rc = lib().tucker_debug_eig(h, d, J, C.c_void_p(S.ctypes.data), C.c_void_p(U.ctypes.data),
                                C.c_void_p(w.ctypes.data))
    _check(rc, h, allow=(E_CONVERGE,))
    return U, w, rc


def tucker_debug_smalldense(mode, A, max_sweeps=30, shift=0.0):
    """mode 0: CholQR factor M of SPD A; mode 1: Jacobi -> (V, theta, sweeps)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    k = A.shape[0]
    out = np.zeros((k, k))
    th = np.zeros(k)
    sw = (C.c_int * 8)()
    _check(lib().tucker_debug_smalldense(mode, k, C.c_void_p(A.ctypes.data), C.c_void_p(out.ctypes.data),
                                         C.c_void_p(th.ctypes.data), C.c_void_p(C.addressof(sw)),
                                         max_sweeps, shift))
    if mode >= 1:
        tucker_debug_smalldense.cycles = list(sw[1:8])
        return out, th, sw[0]
    return out


def tucker_debug_product(S, Y, alpha=1.0, gamma=0.0, D=None):
    """alpha S Y + gamma D on the eigensolver's fp64 tensor-core product."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    d, n = Y.shape
    out = np.zeros((d, n))
    Dp = None
    if D is not None:
        D = np.ascontiguousarray(D, dtype=np.float64)
        Dp = C.c_void_p(D.ctypes.data)
    _check(lib().tucker_debug_product(d, n, C.c_void_p(S.ctypes.data), C.c_void_p(Y.ctypes.data), alpha,
                                      gamma, Dp, C.c_void_p(out.ctypes.data)))
    return out


def tucker_debug_product_time(d, n, reps=50):
    us = C.c_double(0)
    _check(lib().tucker_debug_product_time(d, n, reps, C.byref(us)))
    return us.value


def tucker_csf_stats(h, order=3):
    """Per mode (fibers, nonzeros, virtual fibers, work units) of the HOOI CSF
    orderings; the last two are 0 without a SpTTMc work plan."""
    s = (C.c_int64 * 16)()
    _check(lib().tucker_csf_stats(h, s), h)
    return [tuple(int(s[4 * n + q]) for q in range(4)) for n in range(order)]


def tucker_csf_layout(h, order):
    """Per mode: dict(root, mid0, mid1, leaf, fibers, nodes, nnz, slices) of the CSF
    ordering its HOOI projection uses (mode ids 0-based; mid1 = -1 at order 3)."""
    s = (C.c_int64 * (8 * order))()
    _check(lib().tucker_csf_layout(h, s), h)
    keys = ("root", "mid0", "mid1", "leaf", "fibers", "nodes", "nnz", "slices")
    return [{k: int(s[8 * n + i]) for i, k in enumerate(keys)} for n in range(order)]


def tucker_time_ttmc(h, mode, reps=5):
    """Mean ms of the HOOI projection of `mode` (measurement entry point)."""
    ms = C.c_float(0)
    _check(lib().tucker_time_ttmc(h, mode, reps, C.byref(ms)), h)
    return ms.value


def tucker_mp_overlap_times(h, reset=False):
    """Kernel time (ms) and counts of mp_sweep's overlapped streams since the last reset:
    dict(side_spmm, side_gram, main_spmm, main_gram, eig) -> (ms, count)."""
    ms = (C.c_double * 5)()
    cnt = (C.c_int64 * 5)()
    _check(lib().tucker_mp_overlap_times(h, ms, cnt, 1 if reset else 0), h)
    keys = ("side_spmm", "side_gram", "main_spmm", "main_gram", "eig")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}


def tucker_csf_fibers(h, order=3):
    """Total fibers of the HOOI CSF orderings (all modes)."""
    return sum(st[0] for st in tucker_csf_stats(h, order))


def _run(fn, h, max_sweeps, tol):
    fits = np.zeros(max_sweeps, dtype=np.float64)
    done = C.c_int(0)
    rc = fn(h, max_sweeps, tol, fits.ctypes.data_as(C.POINTER(C.c_double)), C.byref(done))
    _check(rc, h, allow=(E_CONVERGE,))
    return fits[: done.value], rc


def hooi_run(h, max_sweeps=50, tol=1e-4):
    """Sweeps until Delta_fit < tol or max_sweeps (Eq. 10); returns (fits, rc)."""
    return _run(lib().hooi_run, h, max_sweeps, tol)


def mp_run(h, max_sweeps=50, tol=1e-4):
    return _run(lib().mp_run, h, max_sweeps, tol)


def tucker_hosvd(h, mode_mask):
    """U_n <- leading eigenvectors of X_(n) X_(n)^T for the modes in mode_mask."""
    return _check(lib().tucker_hosvd(h, mode_mask), h, allow=(E_CONVERGE,))


def sp_sweep(h, sweeps):
    """Slice Projection sweeps -> (fits, core norms, rc)."""
    fits = np.zeros(sweeps, dtype=np.float64)
    gn = np.zeros(sweeps, dtype=np.float64)
    rc = lib().sp_sweep(h, sweeps, fits.ctypes.data_as(C.POINTER(C.c_double)),
                        gn.ctypes.data_as(C.POINTER(C.c_double)), None)
    _check(rc, h, allow=(E_CONVERGE,))
    return fits, gn, rc


def sp_run(h, max_sweeps=50, tol=1e-4):
    return _run(lib().sp_run, h, max_sweeps, tol)


def tucker_set_factor(h, n, U, check=True):
    if not hasattr(U, "data_ptr"):
        U = np.ascontiguousarray(U, dtype=np.float32)
    if h in _shapes:
        dims, core, dev = _shapes[h]
        if not 0 <= n < len(dims):
            raise ValueError(f"mode {n} out of range for order {len(dims)}")
        _check_array(U, f"U[{n}]", np.float32, shape=(dims[n], core[n]), device=dev)
    _check(lib().tucker_set_factor(h, n, C.c_void_p(_ptr(U)), 1 if check else 0), h)


def _load_torch_nccl():
    """The library dlopens libnccl.so.2 on first use; import torch first so that
    soname resolves to torch's bundled NCCL (a system NCCL loaded first would
    break a later `import torch`, whose libraries need the bundled version)."""
    import torch  # noqa: F401


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (bytes) for tucker_init(..., nccl_id=)."""
    _load_torch_nccl()
    buf = C.create_string_buffer(128)
    _check(lib().tucker_nccl_unique_id(buf))
    return buf.raw


def shard_bounds(work, world):
    """The library's contiguous shard bounds (host only) -> int64 array world+1."""
    w = np.ascontiguousarray(work, dtype=np.float64)
    b = np.zeros(world + 1, dtype=np.int64)
    _check(lib().tucker_shard_bounds(w.ctypes.data_as(C.POINTER(C.c_double)), C.c_int64(w.size),
                                     world, b.ctypes.data_as(C.POINTER(C.c_int64))))
    return b


def tucker_set_allreduce(h, fn):
    """Host collectives: fn(dev_ptr, count, dtype, stream) sums the device buffer
    over the ranks in place (dtype 0 fp32, 1 fp64) and returns 0.  The ctypes
    callback object is returned; keep it alive as long as the handle."""
    cb = ALLREDUCE_FN(lambda p, n, dt, st, user: fn(p, n, dt, st))
    _check(lib().tucker_set_allreduce(h, C.cast(cb, C.c_void_p), None), h)
    return cb


def tucker_shard_info(h, order):
    """This rank's shards: (hooi [(lo, hi)] per mode, mp {(n, m): (lo, hi)})."""
    out = np.zeros(2 * order + 2 * order * order, dtype=np.int64)
    _check(lib().tucker_shard_info(h, out.ctypes.data_as(C.POINTER(C.c_int64))), h)
    hooi = [(int(out[2 * n]), int(out[2 * n + 1])) for n in range(order)]
    mp = {}
    for n in range(order):
        for m in range(order):
            if m != n:
                k = 2 * order + 2 * (n * order + m)
                mp[(n, m)] = (int(out[k]), int(out[k + 1]))
    return hooi, mp


def tucker_stats(h, reset=False):
    s = (C.c_int64 * 18)()
    _check(lib().tucker_stats(h, s, 1 if reset else 0), h)
    names = ("matvec", "reduce", "cholqr", "jacobi", "apply", "deflate", "power", "other")
    return dict(launches=s[0], eig_outer=s[1], eig_matvec=s[2], jacobi_sweeps=s[3],
                gram_path="by-size (dmma <= 2e10 FMA, else tcgen05 3xTF32)" if s[4] == 0 else "all-dmma-fp64",
                eig_phase_ms={n: s[5 + i] / 1e6 for i, n in enumerate(names)},
                eig_flops=s[13],
                product_ms={n: s[14 + i] / 1e6 for i, n in enumerate(("phaseA", "inner_bar", "phaseB", "lead_bar"))})


class Tucker:
    """Convenience wrapper owning one handle."""

    def __init__(self, dims, core, idx, vals, U0, **kw):
        self.dims = tuple(int(x) for x in dims)
        self.core = tuple(int(x) for x in core)
        self.h = tucker_init(self.dims, self.core, idx, vals, U0, **kw)

    def hooi_sweep(self, sweeps, want_stage=False):
        return hooi_sweep(self.h, sweeps, want_stage)

    def mp_sweep(self, sweeps, want_fit=True, want_stage=False):
        return mp_sweep(self.h, sweeps, want_fit, want_stage)

    def core_and_fit(self, **kw):
        return core_and_fit(self.h, self.dims, self.core, **kw)

    def set_factors(self, U):
        tucker_set_factors(self.h, U)

    def debug_ttmc(self, mode):
        P = int(np.prod([J for m, J in enumerate(self.core) if m != mode]))
        return tucker_debug_ttmc(self.h, mode, self.dims[mode], P)

    def sp_sweep(self, sweeps):
        return sp_sweep(self.h, sweeps)

    def sp_run(self, max_sweeps=50, tol=1e-4):
        return sp_run(self.h, max_sweeps, tol)[0]

    def set_factor(self, n, U, check=True):
        tucker_set_factor(self.h, n, U, check)

    def hosvd(self, modes=None):
        """HO-SVD factors for `modes` (default all) into the handle."""
        modes = range(len(self.dims)) if modes is None else modes
        return tucker_hosvd(self.h, sum(1 << m for m in modes))

    def hooi_run(self, max_sweeps=50, tol=1e-4):
        return hooi_run(self.h, max_sweeps, tol)[0]

    def mp_run(self, max_sweeps=50, tol=1e-4):
        return mp_run(self.h, max_sweeps, tol)[0]

    def shard_info(self):
        return tucker_shard_info(self.h, len(self.dims))

    def csf_stats(self):
        return tucker_csf_stats(self.h, len(self.dims))

    def debug_gram(self, algo, mode):
        return tucker_debug_gram(self.h, algo, mode, self.dims[mode])

    def debug_gram_rows(self, algo, mode, rows):
        return tucker_debug_gram_rows(self.h, algo, mode, rows, self.dims[mode])

    def debug_eig(self, S, J):
        return tucker_debug_eig(self.h, S, J)

    def stats(self, reset=False):
        return tucker_stats(self.h, reset)

    def close(self):
        if self.h:
            tucker_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
