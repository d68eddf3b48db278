"""fp64 brute-force CPU oracle for HEGrid's gridding (Eq. 1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2207_04584_b200``) never imports it and shares no
code with it; see ``hegrid_oracle.c`` for the definition it follows and
DESIGN.md "Readings of the paper" for every reading it takes.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(closed forms, invariants, an independent-library neighbour cross-check); none
is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hegrid_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off -fopenmp; no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
             "-shared", "-o", _LIB, _SRC, "-lm"],
            check=True)
    return _LIB


class OraMap(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("crval_lon", ctypes.c_double), ("crval_lat", ctypes.c_double),
                ("crpix_x", ctypes.c_double), ("crpix_y", ctypes.c_double),
                ("cdelt_lon", ctypes.c_double), ("cdelt_lat", ctypes.c_double),
                ("projection", ctypes.c_int32), ("reserved", ctypes.c_int32)]


PROJECTIONS = {"car": 0, "tan": 1, "sin": 2}
_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.ora_grid_cells.argtypes = [P, P, ctypes.c_int64, P, ctypes.c_int64, P, ctypes.c_int64,
                                       ctypes.POINTER(OraMap), ctypes.c_double, ctypes.c_double,
                                       P, ctypes.c_int64, P, P, P, ctypes.c_int, ctypes.c_int]
        lib.ora_grid_cells.restype = ctypes.c_int
        lib.ora_grid_cells_ex.argtypes = lib.ora_grid_cells.argtypes + [P, ctypes.c_int]
        lib.ora_grid_cells_ex.restype = ctypes.c_int
        lib.ora_weight_tophat.argtypes = [ctypes.c_double] * 2
        lib.ora_weight_tophat.restype = ctypes.c_double
        lib.ora_neighbours.argtypes = [P, P, ctypes.c_int64, ctypes.POINTER(OraMap),
                                       ctypes.c_double, ctypes.c_double, P, ctypes.c_int64,
                                       P, P, ctypes.c_int]
        lib.ora_neighbours.restype = ctypes.c_int
        for name in ("ora_distance_deg", "ora_distance_rad"):
            f = getattr(lib, name)
            f.argtypes = [ctypes.c_double] * 4
            f.restype = ctypes.c_double
        lib.ora_weight.argtypes = [ctypes.c_double] * 3
        lib.ora_weight.restype = ctypes.c_double
        lib.ora_sigma_deg.argtypes = [ctypes.c_double]
        lib.ora_sigma_deg.restype = ctypes.c_double
        lib.ora_wrap180.argtypes = [ctypes.c_double]
        lib.ora_wrap180.restype = ctypes.c_double
        lib.ora_cell_centre.argtypes = [ctypes.POINTER(OraMap), ctypes.c_int64, ctypes.c_int64,
                                        ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double)]
        lib.ora_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _map(m) -> OraMap:
    """Accept any object/dict with the hegrid map fields (optional "projection")."""
    g = (lambda k: m[k]) if isinstance(m, dict) else (lambda k: getattr(m, k))
    proj = (m.get("projection", 0) if isinstance(m, dict) else getattr(m, "projection", 0))
    proj = PROJECTIONS[proj] if isinstance(proj, str) else int(proj)
    return OraMap(int(g("nx")), int(g("ny")), float(g("crval_lon")), float(g("crval_lat")),
                  float(g("crpix_x")), float(g("crpix_y")), float(g("cdelt_lon")),
                  float(g("cdelt_lat")), proj, 0)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().ora_max_threads())


def distance_deg(lon1, lat1, lon2, lat2) -> float:
    return float(_load().ora_distance_deg(lon1, lat1, lon2, lat2))


def weight(d_rad, sigma_rad, R_rad) -> float:
    return float(_load().ora_weight(d_rad, sigma_rad, R_rad))


def sigma_deg(fwhm_deg) -> float:
    return float(_load().ora_sigma_deg(fwhm_deg))


def wrap180(x) -> float:
    return float(_load().ora_wrap180(x))


def cell_centre(m, i, j):
    lon, lat = ctypes.c_double(), ctypes.c_double()
    mm = _map(m)
    _load().ora_cell_centre(ctypes.byref(mm), int(i), int(j), ctypes.byref(lon), ctypes.byref(lat))
    return lon.value, lat.value


def grid(lon, lat, vals, m, fwhm_deg, support=3.0, channels=None, cells=None, nthreads=0,
         kernel="gaussian", sample_weights=None, mask=False):
    """Eq. 1 for the given channels (rows of ``vals`` [C][N]) and cells; ``kernel`` is
    "gaussian" (Eq. 1's kernel) or "tophat" (1 inside the support);
    ``sample_weights`` [N] multiply the kernel weight (reading R25); ``mask`` leaves
    non-finite values out of both sums of their channel (reading R24).

    Returns (out [n_ch][n_cells] fp64 with NaN blanks, W [n_cells], nbr_count [n_cells]).
    ``cells`` = linear indices j*nx+i (None = all, in map order).
    """
    lon = np.ascontiguousarray(lon, dtype=np.float64)
    lat = np.ascontiguousarray(lat, dtype=np.float64)
    n = lon.shape[0]
    mm = _map(m)
    if vals is None:
        vals = np.zeros((0, n), np.float32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    if vals.ndim == 1:
        vals = vals[None, :]
    ld = vals.shape[1] if vals.shape[0] else n
    if channels is None:
        ch = None
        n_ch = vals.shape[0]
    else:
        ch = np.ascontiguousarray(channels, dtype=np.int64)
        n_ch = ch.shape[0]
    if cells is None:
        cidx = None
        n_cells = mm.nx * mm.ny
    else:
        cidx = np.ascontiguousarray(cells, dtype=np.int64)
        n_cells = cidx.shape[0]
    out = np.empty((n_ch, n_cells), np.float64)
    W = np.empty(n_cells, np.float64)
    cnt = np.empty(n_cells, np.int64)
    sw = None if sample_weights is None else np.ascontiguousarray(sample_weights, dtype=np.float64)
    if sw is not None and sw.shape != (n,):
        raise ValueError("sample_weights must have one entry per sample")
    rc = _load().ora_grid_cells_ex(_p(lon), _p(lat), n, _p(vals), ld, _p(ch), n_ch,
                                   ctypes.byref(mm), float(fwhm_deg), float(support),
                                   _p(cidx), n_cells, _p(out), _p(W), _p(cnt), int(nthreads),
                                   {"gaussian": 0, "tophat": 1}[kernel], _p(sw), int(bool(mask)))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (code {rc})")
    return out, W, cnt


def neighbours(lon, lat, m, fwhm_deg, support=3.0, cells=None, nthreads=0):
    """CSR neighbour sets (ascending original index): (offsets [n_cells+1], idx)."""
    lon = np.ascontiguousarray(lon, dtype=np.float64)
    lat = np.ascontiguousarray(lat, dtype=np.float64)
    mm = _map(m)
    if cells is None:
        cidx, n_cells = None, mm.nx * mm.ny
    else:
        cidx = np.ascontiguousarray(cells, dtype=np.int64)
        n_cells = cidx.shape[0]
    off = np.zeros(n_cells + 1, np.int64)
    lib = _load()
    rc = lib.ora_neighbours(_p(lon), _p(lat), lon.shape[0], ctypes.byref(mm), float(fwhm_deg),
                            float(support), _p(cidx), n_cells, _p(off), None, int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (code {rc})")
    idx = np.empty(int(off[-1]), np.int64)
    rc = lib.ora_neighbours(_p(lon), _p(lat), lon.shape[0], ctypes.byref(mm), float(fwhm_deg),
                            float(support), _p(cidx), n_cells, _p(off), _p(idx), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (code {rc})")
    return off, idx
