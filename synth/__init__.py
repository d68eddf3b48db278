"""Seeded synthetic inputs shaped like the paper's workloads (shared by tests and bench).

This module holds NONE of the gridding method's arithmetic: no distance, kernel,
bin, sort or normalisation.  It only draws coordinates and sample values, from a
counter-based generator (splitmix64 of (seed, stream, index)) so that any subset
of samples or channels can be regenerated exactly, on CPU or GPU, in any order.

Workload shapes:
  * drift scan (Fig. 1): T tracks of constant dec spread evenly
    over the field, S samples per track evenly spaced in lon with a random per-track
    phase, 0.5 arcsec Gaussian pointing jitter; original order [track][time];
  * uniform random (configs 1 and 3): lon, lat uniform over the field box;
  * values: v[c][n] = 10 + sum_s A_s g_{c,s} exp(-r^2 / 2 sigma_b^2) + 0.1 N(0,1),
    8 compact sources with per-channel spectral weights g, positive baseline
    (shape of SPEC.md:434), fp32 (reading R10: Table 2 sizes imply fp32 values).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict

import torch

# splitmix64 constants as signed int64 (torch has no uint64 arithmetic)
_GOLD = 0x9E3779B97F4A7C15 - (1 << 64)
_M1 = 0xBF58476D1CE4E5B9 - (1 << 64)
_M2 = 0x94D049BB133111EB - (1 << 64)
_K_STREAM = 0xD6E8FEB86659FD93 - (1 << 64)
_MASK53 = (1 << 53) - 1


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 (two's complement) by k."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    z = x + _GOLD
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    return z ^ _srl(z, 31)


def counter_u01(seed: int, stream, index: torch.Tensor) -> torch.Tensor:
    """Uniform [0, 1) doubles indexed by (seed, stream, index)."""
    index = index.to(torch.int64)
    if not torch.is_tensor(stream):
        stream = torch.tensor(int(stream), dtype=torch.int64, device=index.device)
    s = splitmix64(torch.full_like(index, int(seed)) ^ (stream.to(torch.int64) * _K_STREAM))
    z = splitmix64(s ^ splitmix64(index))
    return _srl(z, 11).to(torch.float64) * (1.0 / (1 << 53))


def counter_normal(seed: int, stream, index: torch.Tensor) -> torch.Tensor:
    """Standard normal doubles (Box-Muller on two counter streams)."""
    if torch.is_tensor(stream):
        s0, s1 = 2 * stream, 2 * stream + 1
    else:
        s0, s1 = 2 * int(stream), 2 * int(stream) + 1
    u1 = counter_u01(seed, s0, index)
    u2 = counter_u01(seed, s1, index)
    return torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos((2.0 * math.pi) * u2)


@dataclass
class Workload:
    """One BASELINE.json configuration."""
    name: str
    field_lon: float          # coordinate degrees
    field_lat: float
    n: int
    kind: str                 # "uniform" | "drift"
    nx: int
    ny: int
    cdelt: float              # degrees per cell (both axes)
    channels: int
    fwhm_deg: float           # kernel FWHM
    support: float = 3.0      # R = support * sigma
    centre: tuple = (30.0, 41.0)   # Table 2 map centre, reading R18
    tracks: int = 0           # drift scan: T
    per_track: int = 0        # drift scan: S
    note: str = ""

    @property
    def map(self) -> dict:
        return dict(nx=self.nx, ny=self.ny, crval_lon=self.centre[0], crval_lat=self.centre[1],
                    crpix_x=(self.nx + 1) / 2.0, crpix_y=(self.ny + 1) / 2.0,
                    cdelt_lon=self.cdelt, cdelt_lat=self.cdelt)

    @property
    def cells(self) -> int:
        return self.nx * self.ny

    def with_(self, **kw) -> "Workload":
        d = asdict(self)
        d.update(kw)
        return Workload(**d)


ARCMIN = 1.0 / 60.0

CONFIGS = {
    "cfg1": Workload("cfg1", 1.0, 1.0, 5000, "uniform", 64, 64, 1.0 / 64, 1, 3 * ARCMIN,
                     note="1 ch, 5k random samples, 1x1 deg, 64x64, FWHM 3'"),
    "cfg2": Workload("cfg2", 5.0, 5.0, 1_000_000, "drift", 300, 300, ARCMIN, 256, 3 * ARCMIN,
                     tracks=1000, per_track=1000, note="FAST-like drift scan, 256 ch"),
    "cfg3": Workload("cfg3", 2.0, 2.0, 4_000_000, "uniform", 128, 128, 2.0 / 128, 64,
                     6.925 * ARCMIN, note="high density (~90k neighbours/cell), 64 ch"),
    "cfg4": Workload("cfg4", 5.0, 5.0, 1_000_000, "drift", 300, 300, ARCMIN, 4096, 3 * ARCMIN,
                     tracks=1000, per_track=1000, note="many-channel, 4096 ch"),
    "cfg5": Workload("cfg5", 512 * ARCMIN, 512 * ARCMIN, 2_000_000, "drift", 512, 512, ARCMIN,
                     65536, 3 * ARCMIN, tracks=2000, per_track=1000,
                     note="full FAST width, 65536 ch, streamed"),
    "cfg4s": Workload("cfg4s", 5.0, 5.0, 1_000_000, "drift", 300, 300, ARCMIN, 4096,
                      1.5 * ARCMIN, tracks=1000, per_track=1000,
                      note="sensitivity: half-beam kernel (HBM regime)"),
}

COORD_SEED = 2207
VALUE_SEED = 4584
_CFG_NUM = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4, "cfg5": 5, "cfg4s": 4}


def coord_seed(w: Workload) -> int:
    return COORD_SEED + _CFG_NUM.get(w.name, 0)


def value_seed(w: Workload) -> int:
    return VALUE_SEED + _CFG_NUM.get(w.name, 0)


def coords(w: Workload, seed: int | None = None, device="cpu"):
    """Sample coordinates (lon, lat) in degrees, fp64, original order."""
    seed = coord_seed(w) if seed is None else seed
    lon0, lat0 = w.centre
    if w.kind == "uniform":
        idx = torch.arange(w.n, dtype=torch.int64, device=device)
        lon = lon0 - 0.5 * w.field_lon + w.field_lon * counter_u01(seed, 0, idx)
        lat = lat0 - 0.5 * w.field_lat + w.field_lat * counter_u01(seed, 1, idx)
        return lon, lat
    if w.kind == "drift":
        T, S = w.tracks, w.per_track
        assert T * S == w.n
        t = torch.arange(T, dtype=torch.int64, device=device)
        phase = counter_u01(seed, 2, t)                                   # per-track phase
        dec_t = lat0 - 0.5 * w.field_lat + (t.to(torch.float64) + 0.5) * (w.field_lat / T)
        idx = torch.arange(w.n, dtype=torch.int64, device=device)
        tt, kk = idx // S, idx % S
        lon = lon0 - 0.5 * w.field_lon + (kk.to(torch.float64) + phase[tt]) * (w.field_lon / S)
        lat = dec_t[tt].clone()
        jitter = 0.5 / 3600.0                                             # 0.5 arcsec
        lon = lon + jitter * counter_normal(seed, 3, idx) / math.cos(math.radians(lat0))
        lat = lat + jitter * counter_normal(seed, 4, idx)
        return lon, lat
    raise ValueError(w.kind)


def _sources(w: Workload, seed: int, device):
    k = torch.arange(8, dtype=torch.int64, device=device)
    lon0, lat0 = w.centre
    slon = lon0 + w.field_lon * (counter_u01(seed, 10, k) - 0.5) * 0.8
    slat = lat0 + w.field_lat * (counter_u01(seed, 11, k) - 0.5) * 0.8
    amp = 1.0 + 4.0 * counter_u01(seed, 12, k)
    cen = counter_u01(seed, 13, k) * max(w.channels, 1)
    wid = 1.0 + counter_u01(seed, 14, k) * max(w.channels / 16.0, 1.0)
    return slon, slat, amp, cen, wid


def values(w: Workload, lon: torch.Tensor, lat: torch.Tensor, channels=None, samples=None,
           seed: int | None = None, device=None, dtype=torch.float32) -> torch.Tensor:
    """Sample values [len(channels)][len(samples)] for the given channel ids and
    (original) sample ids.  Any subset regenerates bit-identically."""
    seed = value_seed(w) if seed is None else seed
    device = lon.device if device is None else device
    if channels is None:
        channels = torch.arange(w.channels, dtype=torch.int64, device=device)
    channels = torch.as_tensor(channels, dtype=torch.int64, device=device)
    if samples is None:
        samples = torch.arange(lon.shape[0], dtype=torch.int64, device=device)
    samples = torch.as_tensor(samples, dtype=torch.int64, device=device)
    sl, sb = lon.to(device)[samples], lat.to(device)[samples]
    slon, slat, amp, cen, wid = _sources(w, seed, device)
    sig_b = (3.0 * ARCMIN) / 2.354820045
    cosd0 = math.cos(math.radians(w.centre[1]))
    chf = channels.to(torch.float64)
    out = torch.full((channels.shape[0], samples.shape[0]), 10.0, dtype=torch.float64,
                     device=device)
    for s in range(8):
        prof = torch.exp(-((sl - slon[s]) * cosd0) ** 2 / (2 * sig_b ** 2)
                         - (sb - slat[s]) ** 2 / (2 * sig_b ** 2))         # [n]
        g = 0.2 + torch.exp(-0.5 * ((chf - cen[s]) / wid[s]) ** 2)           # [C]
        out += amp[s] * g[:, None] * prof[None, :]
    noise_idx = channels[:, None] * (1 << 32) + samples[None, :]
    out += 0.1 * counter_normal(seed, 20, noise_idx)
    return out.to(dtype)
