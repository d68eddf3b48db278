"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/hegrid.h declares, and rejects bad arguments before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "hegrid.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(hegrid_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2207_04584_b200 import _binding
    return _binding.load()


def test_header_declares_expected_surface():
    names = _header_functions()
    for n in ("hegrid_plan_create", "hegrid_grid", "hegrid_grid_device", "hegrid_neighbours",
              "hegrid_plan_destroy", "hegrid_status_string"):
        assert n in names


def test_library_exports_every_header_symbol(lib):
    for name in _header_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_binding_covers_every_header_symbol():
    from paper_2207_04584_b200 import _binding
    assert sorted(_binding.SIGNATURES) == _header_functions()


def test_status_strings_and_version(lib):
    from paper_2207_04584_b200 import _binding as b
    assert b.hegrid_abi_version() == 4
    for code in range(7):
        assert len(b.hegrid_status_string(code)) >= 2
    assert "unknown" in b.hegrid_status_string(99)


def test_argument_validation_without_gpu():
    from paper_2207_04584_b200 import _binding as b
    m = dict(nx=8, ny=8, crval_lon=30.0, crval_lat=41.0, crpix_x=4.5, crpix_y=4.5,
             cdelt_lon=1 / 60, cdelt_lat=1 / 60)
    lon = np.array([30.0])
    lat = np.array([41.0])
    with pytest.raises(b.HegridError) as e:
        b.hegrid_plan_create(lon, lat, m, -1.0)
    assert e.value.code == 1
    with pytest.raises(b.HegridError) as e:
        b.hegrid_plan_create(lon, lat, dict(m, nx=0), 0.05)
    assert e.value.code == 1
    with pytest.raises(b.HegridError) as e:
        b.hegrid_plan_create(lon, lat, dict(m, cdelt_lat=0.0), 0.05)
    assert e.value.code == 1
    with pytest.raises(b.HegridError) as e:
        b.hegrid_plan_create(lon, lat, m, 0.05, support_sigma=0.0)
    assert e.value.code == 1
    with pytest.raises(b.HegridError) as e:          # unknown kernel kind
        b.hegrid_plan_create(lon, lat, m, 0.05, kind=7)
    assert e.value.code == 1
    # NULL plan
    assert b.load().hegrid_grid(None, None, 0, None, None) == 1
    assert b.load().hegrid_plan_info(None, None) == 1
    b.hegrid_plan_destroy(None)


def test_no_cpu_fallback_without_gpu():
    """With no device every computing call reports HEGRID_ECUDA instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2207_04584_b200 import _binding as b
    m = dict(nx=8, ny=8, crval_lon=30.0, crval_lat=41.0, crpix_x=4.5, crpix_y=4.5,
             cdelt_lon=1 / 60, cdelt_lat=1 / 60)
    with pytest.raises(b.HegridError) as e:
        b.hegrid_plan_create(np.array([30.0]), np.array([41.0]), m, 0.05)
    assert e.value.code == 4
    with pytest.raises(b.HegridError) as e:
        b.hegrid_sort_u32(np.array([3, 1, 2], np.uint32))
    assert e.value.code == 4


def test_channel_shard_partition():
    from paper_2207_04584_b200 import channel_shard
    for C in (0, 1, 5, 64, 4096, 4099, 65536):
        for G in (1, 2, 3, 4, 8):
            got = [channel_shard(C, G, r) for r in range(G)]
            assert got[0][0] == 0 and got[-1][1] == C
            for (a0, a1), (b0, b1) in zip(got, got[1:]):
                assert a1 == b0 and a0 <= a1
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 4
