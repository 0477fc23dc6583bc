"""Host-side checks of the C-ABI library (no GPU needed): it builds/loads,
exports every symbol include/tucker.h declares, and rejects bad arguments
before touching the device."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "tucker.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_0711_2023_b200 import capi
    if not os.path.exists(capi.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return capi.lib()


def test_header_symbols_exported(lib):
    from paper_0711_2023_b200 import capi
    names = _header_functions()
    assert len(names) >= 13
    assert sorted(capi.EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n


def test_strerror_and_arg_errors_without_device(lib):
    from paper_0711_2023_b200 import capi
    assert lib.tucker_strerror(0) == b"ok"
    assert lib.tucker_strerror(3) == b"duplicate coordinate"
    dims, core = (4, 5, 6), (2, 2, 2)
    idx = [np.zeros(3, np.int32)] * 3
    vals = np.ones(3, np.float32)
    U = [np.eye(d, c, dtype=np.float32) for d, c in zip(dims, core)]
    # orders outside 2..8 (HOOI's range) -> E_ARG before any CUDA call; orders 2 and
    # 5..8 run HOOI on one rank only (gen.cu): sharded -> E_ARG
    d9 = (4, 5, 6, 7, 8, 4, 5, 6, 7)
    U9 = [np.eye(d, 2, dtype=np.float32) for d in d9]
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(d9, (2,) * 9, (idx * 3)[:9], vals, U9)
    assert e.value.code == 1
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init((4,), (2,), idx[:1], vals, [np.eye(4, 2, dtype=np.float32)])
    assert e.value.code == 1
    d5 = (4, 5, 6, 7, 8)
    U5 = [np.eye(d, 2, dtype=np.float32) for d in d5]
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(d5, (2,) * 5, (idx * 2)[:5], vals, U5, rank=0, world=2, host_collectives=True)
    assert e.value.code == 1
    # J > I -> E_ARG
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(dims, (5, 2, 2), idx, vals, [np.eye(4, 5, dtype=np.float32)] + U[1:])
    assert e.value.code == 1
    # non-orthonormal initial factor -> E_FACTOR (host check)
    Ubad = [u.copy() for u in U]
    Ubad[1][0, 0] = 2.0
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(dims, core, idx, vals, Ubad)
    assert e.value.code == 5


def test_new_entry_points_reject_bad_arguments_without_device(lib):
    """The drivers, HO-SVD, Slice Projection, factor setter and multi-GPU
    helpers validate their arguments before any device work (E_ARG = 1)."""
    import ctypes as C
    from paper_0711_2023_b200 import capi
    d = C.c_double(0)
    i = C.c_int(0)
    nul = None
    assert lib.hooi_run(nul, 5, 1e-4, C.byref(d), C.byref(i)) == 1
    assert lib.mp_run(nul, 5, 1e-4, C.byref(d), C.byref(i)) == 1
    assert lib.sp_run(nul, 5, 1e-4, C.byref(d), C.byref(i)) == 1
    assert lib.sp_sweep(nul, 1, None, None, None) == 1
    assert lib.tucker_hosvd(nul, 1) == 1
    assert lib.tucker_set_factor(nul, 0, nul, 1) == 1
    assert lib.tucker_shard_info(nul, nul) == 1
    assert lib.tucker_nccl_unique_id(nul) == 1
    b = np.zeros(3, np.int64)
    w = np.ones(4)
    bp = b.ctypes.data_as(C.POINTER(C.c_int64))
    wp = w.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.tucker_shard_bounds(wp, 4, 0, bp) == 1   # world < 1
    assert lib.tucker_shard_bounds(wp, -1, 2, bp) == 1  # n < 0
    assert lib.tucker_shard_bounds(None, 4, 2, bp) == 1
    # world > 1 without an NCCL id, and rank outside [0, world): E_ARG before any CUDA call
    dims, core = (4, 5, 6), (2, 2, 2)
    idx = [np.zeros(3, np.int32)] * 3
    vals = np.ones(3, np.float32)
    U = [np.eye(n, c, dtype=np.float32) for n, c in zip(dims, core)]
    for kw in ({"world": 2}, {"rank": 2, "world": 2, "nccl_id": b"\0" * 128}, {"rank": -1}):
        with pytest.raises(capi.TuckerError) as e:
            capi.tucker_init(dims, core, idx, vals, U, **kw)
        assert e.value.code == 1, kw


def test_binding_checks_sizes_before_the_c_call(lib):
    """the C side copies nnz / I_n x J_n elements from the caller's
    pointers, so the binding rejects short or mis-shaped arrays first."""
    from paper_0711_2023_b200 import capi
    dims, core = (4, 5, 6), (2, 2, 2)
    idx = [np.zeros(3, np.int32)] * 3
    vals = np.ones(3, np.float32)
    U = [np.eye(d, c, dtype=np.float32) for d, c in zip(dims, core)]
    with pytest.raises(ValueError, match="idx\\[1\\]"):
        capi.tucker_init(dims, core, [idx[0], np.zeros(2, np.int32), idx[2]], vals, U)
    with pytest.raises(ValueError, match="U0\\[2\\]"):
        capi.tucker_init(dims, core, idx, vals, U[:2] + [np.eye(5, 2, dtype=np.float32)])
    with pytest.raises(ValueError, match="need 3"):
        capi.tucker_init(dims, core, idx[:2], vals, U)


def test_init_rejects_key_overflow_and_oversized_core(lib):
    """a tensor whose dims multiply past 2^64 cannot be packed into
    the CSF sort keys; J_n > prod_{q != n} J_q has no J_n-dimensional dominant
    subspace of Y_(n).  Both are E_ARG before any device work."""
    from paper_0711_2023_b200 import capi
    dims = (3_000_000, 2_000_000, 2_000_000_000 - 1)  # ~1.2e22 > 2^64
    core = (2, 2, 2)
    idx = [np.zeros(1, np.int32)] * 3
    U = [np.zeros((d, c), np.float32) for d, c in zip(dims[:2], core[:2])]
    # factors of the huge mode would not fit in host memory: pass a tiny stand-in through the C call
    import ctypes as C
    o = capi.tucker_opts()
    lib.tucker_default_opts(C.byref(o))
    u_small = np.zeros(4, np.float32)
    d = (C.c_int64 * 3)(*dims)
    j = (C.c_int64 * 3)(*core)
    ip = (C.c_void_p * 3)(*[a.ctypes.data for a in idx])
    up = (C.c_void_p * 3)(*([u_small.ctypes.data] * 3))
    h = C.c_void_p()
    o.flags = capi.TUCKER_INPUT_ON_DEVICE  # skip the host orthonormality check of the stand-in
    vals = np.ones(1, np.float32)
    assert lib.tucker_init(C.byref(h), 3, d, j, 1, ip, C.c_void_p(vals.ctypes.data), up, C.byref(o)) == 1
    dims, core = (10, 10, 10), (9, 2, 4)  # J_1 = 9 > J_2 J_3 = 8
    idx = [np.zeros(3, np.int32)] * 3
    U = [np.eye(n, c, dtype=np.float32) for n, c in zip(dims, core)]
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(dims, core, idx, np.ones(3, np.float32), U)
    assert e.value.code == 1
