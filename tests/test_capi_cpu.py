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
    # order 5 is outside the paper's MP scope (reading A18) -> E_ARG before any CUDA call
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init((4, 5, 6, 7, 8), (2,) * 5, (idx * 2)[:5], vals, (U * 2)[:5])
    assert e.value.code == 1
    # J > I -> E_ARG
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(dims, (5, 2, 2), idx, vals, U)
    assert e.value.code == 1
    # non-orthonormal initial factor -> E_FACTOR (host check)
    Ubad = [u.copy() for u in U]
    Ubad[1][0, 0] = 2.0
    with pytest.raises(capi.TuckerError) as e:
        capi.tucker_init(dims, core, idx, vals, Ubad)
    assert e.value.code == 5
