"""C-ABI library: loads on CPU, exports every symbol include/metro_route.h declares,
host-side helpers behave (no compute calls -- those need a GPU)."""

import ctypes

import numpy as np
import pytest

from paper_2512_09277_b200 import _native


def test_library_loads_and_exports_header_symbols():
    L = _native.lib()
    names = _native.exported_symbols()
    assert len(names) >= 14
    for name in names:
        assert hasattr(L, name), name
    assert L.metro_abi_version() == _native.ABI_VERSION


def test_header_symbols_match_nm():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(_native.exported_symbols()) <= exported


def test_strerror_and_mask_words():
    L = _native.lib()
    assert L.metro_strerror(0) == b"ok"
    assert b"binary" in L.metro_strerror(_native.ENOTBINARY)
    assert [L.metro_mask_words(g) for g in (1, 32, 33, 64, 65, 128)] == [1, 1, 2, 2, 3, 4]


def test_pack_placement_host():
    from paper_2512_09277_b200 import pack_placement, ValidationError

    A = np.zeros((3, 40), dtype=np.int8)
    A[0, [0, 5, 31]] = 1
    A[1, [32, 39]] = 1
    A[2, 7] = 1
    m = pack_placement(A)
    assert m.shape == (3, 2)
    assert m[0, 0] == (1 | (1 << 5) | (1 << 31)) and m[0, 1] == 0
    assert m[1, 0] == 0 and m[1, 1] == (1 | (1 << 7))
    assert m[2, 0] == 1 << 7
    with pytest.raises(ValidationError, match="binary"):
        pack_placement(np.array([[2, 0]]))


def test_host_workspace_bytes():
    L = _native.lib()
    assert L.metro_host_workspace_bytes(8192, 256, 8) >= 8192 * 4 * 2 + (8 + 8 + 256) * 4


def test_argument_errors_without_gpu():
    """Host-side validation returns before any CUDA call."""
    L = _native.lib()
    assert L.metro_route_v1(None, 0, None, 4, 2, None, None, None, None, None, None, 0, None) == _native.EARG
    dummy = ctypes.c_void_p(1)
    assert L.metro_route_v1(dummy, 8, dummy, 4, 200, None, dummy, dummy, dummy, None, dummy, 0, None) == _native.EDIMS
    assert L.metro_route_v1(dummy, 8, dummy, 0, 2, None, dummy, dummy, dummy, None, dummy, 0, None) == _native.EDIMS
    assert L.metro_route_v1(dummy, 8, dummy, 4, 2, None, dummy, dummy, dummy, None, dummy, 3, None) == _native.EARG
