"""Thin ctypes binding of include/hegrid.h (argument marshalling only).

Every numeric step runs inside libhegrid.so's sm_100a kernels; this module only
converts Python/numpy/torch arguments to pointers and status codes to exceptions.
There is no CPU fallback: importing fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEGRID_LIB") or os.path.join(_HERE, "libhegrid.so")

HEGRID_OK = 0
STATUS = {0: "HEGRID_OK", 1: "HEGRID_EINVAL", 2: "HEGRID_EDOMAIN", 3: "HEGRID_ENOMEM",
          4: "HEGRID_ECUDA", 5: "HEGRID_EUNSUPPORTED", 6: "HEGRID_EINTERNAL"}
HEGRID_LAYOUT_USER_CN = 0
HEGRID_LAYOUT_PLAN_NC = 1
HEGRID_ENGINE_AUTO = 0
HEGRID_ENGINE_SIMT = 1
HEGRID_ENGINE_TC = 2


class HegridError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)} ({_status_string(code)})")


class hegrid_map(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("crval_lon", ctypes.c_double), ("crval_lat", ctypes.c_double),
                ("crpix_x", ctypes.c_double), ("crpix_y", ctypes.c_double),
                ("cdelt_lon", ctypes.c_double), ("cdelt_lat", ctypes.c_double),
                ("projection", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class hegrid_kernel(ctypes.Structure):
    _fields_ = [("fwhm_deg", ctypes.c_double), ("support_sigma", ctypes.c_double),
                ("kind", ctypes.c_int32), ("reserved", ctypes.c_int32)]


HEGRID_KERNEL_GAUSSIAN, HEGRID_KERNEL_TOPHAT = 0, 1
KERNELS = {"gaussian": HEGRID_KERNEL_GAUSSIAN, "tophat": HEGRID_KERNEL_TOPHAT}


class hegrid_opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("n_streams", ctypes.c_int32),
                ("channel_block", ctypes.c_int32), ("engine", ctypes.c_int32),
                ("weight_image_max_bytes", ctypes.c_int64), ("index", ctypes.c_int32),
                ("nonfinite", ctypes.c_int32)]


class hegrid_plan_stats(ctypes.Structure):
    _fields_ = [("n_samples", ctypes.c_int64), ("n_used", ctypes.c_int64),
                ("n_bins", ctypes.c_int64), ("n_candidate_pairs", ctypes.c_int64),
                ("n_pairs", ctypes.c_int64), ("nbr_min", ctypes.c_int32),
                ("nbr_max", ctypes.c_int32), ("nbr_mean", ctypes.c_double),
                ("t_plan_ms", ctypes.c_double), ("nrow", ctypes.c_int32),
                ("ncol", ctypes.c_int32), ("mlat", ctypes.c_int32), ("mlon", ctypes.c_int32),
                ("sigma_deg", ctypes.c_double), ("radius_deg", ctypes.c_double),
                ("weight_image_bytes", ctypes.c_int64), ("tc_entries", ctypes.c_int64),
                ("tc_block_slots", ctypes.c_int64), ("index", ctypes.c_int32),
                ("nside", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
PLAN = ctypes.c_void_p

# name -> (restype, argtypes); the C-ABI surface, one entry per declaration in hegrid.h
SIGNATURES = {
    "hegrid_plan_create": (I32, [P, P, I64, ctypes.POINTER(hegrid_map),
                                 ctypes.POINTER(hegrid_kernel), ctypes.POINTER(hegrid_opts),
                                 ctypes.POINTER(PLAN)]),
    "hegrid_plan_create_device": (I32, [P, P, I64, ctypes.POINTER(hegrid_map),
                                        ctypes.POINTER(hegrid_kernel), ctypes.POINTER(hegrid_opts),
                                        P, ctypes.POINTER(PLAN)]),
    "hegrid_plan_destroy": (None, [PLAN]),
    "hegrid_plan_info": (I32, [PLAN, ctypes.POINTER(hegrid_plan_stats)]),
    "hegrid_plan_permutation": (I32, [PLAN, P, P]),
    "hegrid_grid": (I32, [PLAN, P, I64, P, P]),
    "hegrid_grid_device": (I32, [PLAN, P, I64, I64, I32, P, P, P]),
    "hegrid_permute_device": (I32, [PLAN, P, I64, I64, P, I64, P]),
    "hegrid_neighbours": (I32, [PLAN, I64, I64, P, P]),
    "hegrid_sort_u32": (I32, [P, I64, P, I32]),
    "hegrid_healpix_ang2pix": (I32, [I32, P, P, I64, P, I32]),
    "hegrid_plan_set_sample_weights": (I32, [PLAN, P, I64]),
    "hegrid_profile_enable": (I32, [PLAN, I32]),
    "hegrid_profile_read": (I32, [PLAN, P, P]),
    "hegrid_pipeline_trace": (I32, [PLAN, P, I64, P]),
    "hegrid_launch_count": (I64, []),
    "hegrid_status_string": (ctypes.c_char_p, [I32]),
    "hegrid_abi_version": (I32, []),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libhegrid.so (raises if it is not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(the hegrid CUDA library has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _status_string(code: int) -> str:
    try:
        return load().hegrid_status_string(code).decode()
    except Exception:
        return "?"


def _check(code: int, where: str):
    if code != HEGRID_OK:
        raise HegridError(code, where)


def _ptr(x):
    """Pointer of a numpy array, torch tensor, int address or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError(type(x))


PROJECTIONS = {"car": 0, "tan": 1, "sin": 2}


def make_map(m) -> hegrid_map:
    g = (lambda k: m[k]) if isinstance(m, dict) else (lambda k: getattr(m, k))
    proj = (m.get("projection", 0) if isinstance(m, dict) else getattr(m, "projection", 0))
    proj = PROJECTIONS[proj] if isinstance(proj, str) else int(proj)
    return hegrid_map(int(g("nx")), int(g("ny")), float(g("crval_lon")), float(g("crval_lat")),
                      float(g("crpix_x")), float(g("crpix_y")), float(g("cdelt_lon")),
                      float(g("cdelt_lat")), proj, 0)


HEGRID_INDEX_AUTO, HEGRID_INDEX_BINS, HEGRID_INDEX_HEALPIX = 0, 1, 2
INDEXES = {"auto": HEGRID_INDEX_AUTO, "bins": HEGRID_INDEX_BINS, "healpix": HEGRID_INDEX_HEALPIX}


HEGRID_NONFINITE_PROPAGATE, HEGRID_NONFINITE_MASK = 0, 1
NONFINITE = {"propagate": HEGRID_NONFINITE_PROPAGATE, "mask": HEGRID_NONFINITE_MASK}


def make_opts(device=0, n_streams=0, channel_block=0, engine=0,
              weight_image_max_bytes=0, index=HEGRID_INDEX_AUTO,
              nonfinite=HEGRID_NONFINITE_PROPAGATE) -> hegrid_opts:
    return hegrid_opts(device, n_streams, channel_block, engine, weight_image_max_bytes, index,
                       nonfinite)


# ----------------------------------------------------------------- C-ABI names
def hegrid_plan_create(lon_deg: np.ndarray, lat_deg: np.ndarray, m, fwhm_deg: float,
                       support_sigma: float = 3.0, opts: hegrid_opts | None = None,
                       kind: int = HEGRID_KERNEL_GAUSSIAN) -> int:
    lon = np.ascontiguousarray(lon_deg, np.float64)
    lat = np.ascontiguousarray(lat_deg, np.float64)
    if lon.shape != lat.shape or lon.ndim != 1:
        raise ValueError("lon/lat must be equal-length 1-D arrays")
    mm, kk = make_map(m), hegrid_kernel(fwhm_deg, support_sigma, kind, 0)
    out = PLAN()
    _check(load().hegrid_plan_create(_ptr(lon), _ptr(lat), lon.shape[0], ctypes.byref(mm),
                                     ctypes.byref(kk), ctypes.byref(opts) if opts else None,
                                     ctypes.byref(out)), "hegrid_plan_create")
    return out.value


def hegrid_plan_create_device(d_lon, d_lat, n: int, m, fwhm_deg: float,
                              support_sigma: float = 3.0, opts: hegrid_opts | None = None,
                              stream: int = 0, kind: int = HEGRID_KERNEL_GAUSSIAN) -> int:
    mm, kk = make_map(m), hegrid_kernel(fwhm_deg, support_sigma, kind, 0)
    out = PLAN()
    _check(load().hegrid_plan_create_device(_ptr(d_lon), _ptr(d_lat), n, ctypes.byref(mm),
                                            ctypes.byref(kk),
                                            ctypes.byref(opts) if opts else None, stream,
                                            ctypes.byref(out)), "hegrid_plan_create_device")
    return out.value


def hegrid_plan_destroy(plan: int) -> None:
    load().hegrid_plan_destroy(plan)


def hegrid_plan_info(plan: int) -> dict:
    st = hegrid_plan_stats()
    _check(load().hegrid_plan_info(plan, ctypes.byref(st)), "hegrid_plan_info")
    return st.as_dict()


def hegrid_plan_permutation(plan: int) -> np.ndarray:
    n_used = ctypes.c_int64()
    _check(load().hegrid_plan_permutation(plan, None, ctypes.addressof(n_used)),
           "hegrid_plan_permutation")
    perm = np.empty(n_used.value, np.int64)
    _check(load().hegrid_plan_permutation(plan, _ptr(perm), None), "hegrid_plan_permutation")
    return perm


def hegrid_grid(plan: int, data, n_channels: int, out_map, weight_map=None) -> None:
    _check(load().hegrid_grid(plan, _ptr(data), n_channels, _ptr(out_map), _ptr(weight_map)),
           "hegrid_grid")


def hegrid_grid_device(plan: int, d_data, n_channels: int, ld: int, layout: int, d_out,
                       d_weight=None, stream: int = 0) -> None:
    _check(load().hegrid_grid_device(plan, _ptr(d_data), n_channels, ld, layout, _ptr(d_out),
                                     _ptr(d_weight), stream), "hegrid_grid_device")


def hegrid_permute_device(plan: int, d_user, n_channels: int, ld_user: int, d_plan,
                          ld_plan: int, stream: int = 0) -> None:
    _check(load().hegrid_permute_device(plan, _ptr(d_user), n_channels, ld_user, _ptr(d_plan),
                                        ld_plan, stream), "hegrid_permute_device")


def hegrid_neighbours(plan: int, cell_begin: int, cell_end: int):
    off = np.zeros(cell_end - cell_begin + 1, np.int64)
    _check(load().hegrid_neighbours(plan, cell_begin, cell_end, _ptr(off), None),
           "hegrid_neighbours")
    idx = np.empty(int(off[-1]), np.int64)
    _check(load().hegrid_neighbours(plan, cell_begin, cell_end, _ptr(off), _ptr(idx)),
           "hegrid_neighbours")
    return off, idx


def hegrid_sort_u32(keys: np.ndarray, device: int = 0) -> np.ndarray:
    k = np.ascontiguousarray(keys, np.uint32)
    perm = np.empty(k.shape[0], np.int32)
    _check(load().hegrid_sort_u32(_ptr(k), k.shape[0], _ptr(perm), device), "hegrid_sort_u32")
    return perm


def hegrid_plan_set_sample_weights(plan: int, omega) -> None:
    """Per-sample weights (original sample order) multiplying the kernel weight; None = 1."""
    if omega is None:
        _check(load().hegrid_plan_set_sample_weights(plan, None, 0), "hegrid_plan_set_sample_weights")
        return
    w = np.ascontiguousarray(omega, np.float32)
    _check(load().hegrid_plan_set_sample_weights(plan, _ptr(w), w.shape[0]), "hegrid_plan_set_sample_weights")


def hegrid_healpix_ang2pix(nside: int, theta: np.ndarray, phi: np.ndarray, device: int = 0) -> np.ndarray:
    """Ring-scheme pixel of each (colatitude, longitude) in radians, on the device."""
    t = np.ascontiguousarray(theta, np.float64)
    f = np.ascontiguousarray(phi, np.float64)
    if t.shape != f.shape or t.ndim != 1:
        raise ValueError("theta/phi must be equal-length 1-D arrays")
    pix = np.empty(t.shape[0], np.int64)
    _check(load().hegrid_healpix_ang2pix(nside, _ptr(t), _ptr(f), t.shape[0], _ptr(pix), device),
           "hegrid_healpix_ang2pix")
    return pix


def hegrid_profile_enable(plan: int, enable: bool = True) -> None:
    _check(load().hegrid_profile_enable(plan, int(bool(enable))), "hegrid_profile_enable")


def hegrid_profile_read(plan: int):
    ms = ctypes.c_double()
    k = ctypes.c_int64()
    _check(load().hegrid_profile_read(plan, ctypes.addressof(ms), ctypes.addressof(k)),
           "hegrid_profile_read")
    return ms.value, k.value


def hegrid_pipeline_trace(plan: int) -> np.ndarray:
    """[blocks][5] rows {slot, h2d_start, h2d_end, compute_end, d2h_end} (ms)."""
    n = ctypes.c_int64()
    _check(load().hegrid_pipeline_trace(plan, None, 0, ctypes.addressof(n)), "hegrid_pipeline_trace")
    buf = np.zeros((n.value, 5), np.float64)
    _check(load().hegrid_pipeline_trace(plan, _ptr(buf), n.value, ctypes.addressof(n)),
           "hegrid_pipeline_trace")
    return buf


def hegrid_launch_count() -> int:
    return int(load().hegrid_launch_count())


def hegrid_status_string(code: int) -> str:
    return load().hegrid_status_string(code).decode()


def hegrid_abi_version() -> int:
    return int(load().hegrid_abi_version())
