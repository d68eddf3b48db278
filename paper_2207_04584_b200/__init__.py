"""HEGrid hot path on B200: convolution gridding of many-channel single-dish spectra.

Python face of the C ABI in include/hegrid.h (``_binding`` re-exports the same names).
``Plan`` is a convenience wrapper that marshals numpy / torch arguments; every numeric
step runs in libhegrid.so's sm_100a kernels (no CPU fallback).
"""
from __future__ import annotations

import numpy as np

from . import _binding as abi
from ._binding import (HEGRID_ENGINE_TC, HEGRID_LAYOUT_PLAN_NC, HEGRID_LAYOUT_USER_CN, HegridError,  # noqa: F401
                       KERNELS, hegrid_abi_version, hegrid_grid, hegrid_grid_device,
                       hegrid_launch_count, hegrid_neighbours, hegrid_permute_device,
                       hegrid_plan_create, hegrid_plan_create_device, hegrid_plan_destroy,
                       hegrid_pipeline_trace, hegrid_plan_info, hegrid_plan_permutation,
                       hegrid_profile_enable,
                       hegrid_profile_read, hegrid_sort_u32, hegrid_status_string, make_map,
                       make_opts, hegrid_healpix_ang2pix, hegrid_plan_set_sample_weights, INDEXES,
                       NONFINITE)
from .shard import channel_shard  # noqa: F401

__all__ = ["Plan", "abi", "channel_shard", "HegridError"]


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """Spatial index + geometry shared by every channel.

    lon, lat: degrees, numpy / CPU tensors (host plan build) or CUDA tensors (device
    build).  ``map``: dict with nx, ny, crval_lon, crval_lat, crpix_x, crpix_y,
    cdelt_lon, cdelt_lat.
    """

    ENGINES = {"auto": 0, "simt": 1, "tc": 2}

    def __init__(self, lon, lat, map, fwhm_deg, support_sigma=3.0, device=0, n_streams=0,
                 channel_block=0, stream=None, engine="auto", kernel="gaussian",
                 weight_image_max_bytes=0, index="auto", nonfinite="propagate"):
        self.map = dict(map) if isinstance(map, dict) else map
        self.nx, self.ny = int(self.map["nx"]), int(self.map["ny"])
        self.device = device
        opts = make_opts(device, n_streams, channel_block, self.ENGINES[engine],
                         weight_image_max_bytes, INDEXES[index], NONFINITE[nonfinite])
        if hasattr(lon, "is_cuda") and lon.is_cuda:
            import torch
            lon = lon.to(torch.float64).contiguous()
            lat = lat.to(torch.float64).contiguous()
            self.n = lon.shape[0]
            self._h = hegrid_plan_create_device(lon, lat, self.n, self.map, fwhm_deg,
                                                support_sigma, opts, _stream_handle(stream),
                                                KERNELS[kernel])
        else:
            lon = np.ascontiguousarray(np.asarray(lon), np.float64)
            lat = np.ascontiguousarray(np.asarray(lat), np.float64)
            self.n = lon.shape[0]
            self._h = hegrid_plan_create(lon, lat, self.map, fwhm_deg, support_sigma, opts,
                                         KERNELS[kernel])

    # -------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_h", None):
            hegrid_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self) -> int:
        return self._h

    @property
    def cells(self) -> int:
        return self.nx * self.ny

    # -------------------------------------------------------------- queries
    def info(self) -> dict:
        return hegrid_plan_info(self._h)

    def set_sample_weights(self, omega):
        """Per-sample weights omega[n] >= 0 (original order) multiplying the kernel weight
        (hegrid_plan_set_sample_weights); None restores 1."""
        if omega is not None and hasattr(omega, "detach"):
            omega = omega.detach().cpu().numpy()
        hegrid_plan_set_sample_weights(self._h, omega)

    def permutation(self) -> np.ndarray:
        return hegrid_plan_permutation(self._h)

    def neighbours(self, cell_begin=0, cell_end=None):
        return hegrid_neighbours(self._h, cell_begin, self.cells if cell_end is None else cell_end)

    # -------------------------------------------------------------- gridding
    def grid(self, data, out=None, weight=None, stream=None):
        """Eq. 1 for data [C][N] (original sample order).

        numpy / CPU tensor -> host end-to-end path (hegrid_grid), returns numpy/tensor
        out [C][ny][nx] and weight [ny][nx] on the host; CUDA tensor -> device path
        (hegrid_grid_device, USER_CN layout) on ``stream``.
        """
        if hasattr(data, "is_cuda") and data.is_cuda:
            import torch
            C = data.shape[0]
            assert data.dtype == torch.float32 and data.stride(1) == 1
            if out is None:
                out = torch.empty((C, self.ny, self.nx), dtype=torch.float32, device=data.device)
            if weight is None:
                weight = torch.empty((self.ny, self.nx), dtype=torch.float32, device=data.device)
            hegrid_grid_device(self._h, data, C, data.stride(0), HEGRID_LAYOUT_USER_CN, out,
                               weight, _stream_handle(stream))
            return out, weight
        is_torch = hasattr(data, "data_ptr")
        if is_torch:
            import torch
            assert data.dtype == torch.float32 and data.is_contiguous()
            C = data.shape[0]
            if out is None:
                out = torch.empty((C, self.ny, self.nx), dtype=torch.float32)
            if weight is None:
                weight = torch.empty((self.ny, self.nx), dtype=torch.float32)
        else:
            data = np.ascontiguousarray(data, np.float32)
            if data.ndim == 1:
                data = data[None]
            C = data.shape[0]
            if out is None:
                out = np.empty((C, self.ny, self.nx), np.float32)
            if weight is None:
                weight = np.empty((self.ny, self.nx), np.float32)
        hegrid_grid(self._h, data, C, out, weight)
        return out, weight

    def grid_plan_layout(self, v_plan, n_channels, out, weight=None, stream=None):
        """Device hot path on plan-ordered, channel-contiguous values v_plan [n_used][ld]."""
        hegrid_grid_device(self._h, v_plan, n_channels, v_plan.stride(0), HEGRID_LAYOUT_PLAN_NC,
                           out, weight, _stream_handle(stream))
        return out, weight

    def permute(self, d_user, d_plan, stream=None):
        """Device permute of user-order [C][N] values into plan layout [n_used][ld]."""
        hegrid_permute_device(self._h, d_user, d_user.shape[0], d_user.stride(0), d_plan,
                              d_plan.stride(0), _stream_handle(stream))
        return d_plan

    def profile(self, enable=True):
        hegrid_profile_enable(self._h, enable)

    def profile_read(self):
        return hegrid_profile_read(self._h)

    def pipeline_trace(self):
        """Per-block stage times of the last profiled host grid call (hegrid_pipeline_trace)."""
        return hegrid_pipeline_trace(self._h)
