"""BASELINE.json's synthetic scene generator (stands in for the paper's AVIRIS cubes).

Background pixel = sum_j alpha_j e_j(b) + N(0, 0.01^2) with alpha ~ Dirichlet(1) over
5 endmembers; each endmember is a sum of 3 Gaussian bumps over the band index,
e(b) = sum_m a_m exp(-((b - c_m)/w_m)^2) with c ~ U[0, L), w ~ U[5, 40], a ~ U[0.1, 1]
(the bump shape of the reference's `peaks` spectra, proj/core/src/synth.cpp:234-247,
taken over the band index). Anomalies: `rate` of the pixels, in clusters of 1-3
pixels, blend a 6th endmember, z = (1 - f) b + f e6 with f ~ U[0.3, 1.0] (the
Eq. 10 sub-pixel model, proj/core/src/synth.cpp:20-27); the truth mask marks the
cluster pixels. fp32 BIP output.

Rows are generated in fixed 64-row chunks, each from its own seeded torch
generator, so any row range (a rank's strip + halo) is reproduced byte for byte
on the same device type, independent of how the image is split.
"""
from __future__ import annotations

import math

import torch

CHUNK = 64


def endmembers(bands: int, seed: int) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    p = torch.rand((6, 3, 3), generator=g, dtype=torch.float64)
    c = p[..., 0] * bands
    w = 5.0 + 35.0 * p[..., 1]
    a = 0.1 + 0.9 * p[..., 2]
    b = torch.arange(bands, dtype=torch.float64)
    e = (a[..., None] * torch.exp(-(((b - c[..., None]) / w[..., None]) ** 2))).sum(1)
    return e  # (6, bands)


def anomaly_plan(lines: int, samples: int, rate: float, seed: int):
    """Cluster pixels (row, col) and their fill fractions, plus the truth mask."""
    g = torch.Generator().manual_seed(seed ^ 0x5EED)
    npix = lines * samples
    n_clusters = max(1, int(round(rate * npix / 2.0)))
    rows = torch.randint(0, lines, (n_clusters,), generator=g)
    cols = torch.randint(0, samples, (n_clusters,), generator=g)
    sizes = torch.randint(1, 4, (n_clusters,), generator=g)
    fracs = 0.3 + 0.7 * torch.rand((n_clusters,), generator=g, dtype=torch.float64)
    truth = torch.zeros((lines, samples), dtype=torch.uint8)
    fill = torch.zeros((lines, samples), dtype=torch.float64)
    offsets = [(0, 0), (0, 1), (1, 0)]
    for r, c, s, f in zip(rows.tolist(), cols.tolist(), sizes.tolist(), fracs.tolist()):
        for dr, dc in offsets[:s]:
            rr, cc = r + dr, c + dc
            if rr < lines and cc < samples:
                truth[rr, cc] = 1
                fill[rr, cc] = f
    return truth, fill


def generate_rows(lines: int, samples: int, bands: int, seed: int, row0: int, row1: int,
                  rate: float = 0.002, device="cpu", noise: float = 0.01) -> torch.Tensor:
    """Rows [row0, row1) of the scene as an fp32 (rows, samples, bands) tensor."""
    e = endmembers(bands, seed).to(device=device, dtype=torch.float32)
    _, fill = anomaly_plan(lines, samples, rate, seed)
    out = torch.empty((row1 - row0, samples, bands), dtype=torch.float32, device=device)
    k0, k1 = row0 // CHUNK, (row1 + CHUNK - 1) // CHUNK
    for k in range(k0, k1):
        a, b = k * CHUNK, min((k + 1) * CHUNK, lines)
        g = torch.Generator(device=device).manual_seed(seed * 1_000_003 + k + 1)
        u = torch.rand((b - a, samples, 5), generator=g, device=device, dtype=torch.float32)
        alpha = -torch.log(u.clamp_min(1e-12))
        alpha = alpha / alpha.sum(-1, keepdim=True)
        bg = alpha @ e[:5]
        bg += noise * torch.randn((b - a, samples, bands), generator=g, device=device,
                                  dtype=torch.float32)
        f = fill[a:b].to(device=device, dtype=torch.float32)[..., None]
        bg = (1.0 - f) * bg + f * e[5]
        lo, hi = max(a, row0), min(b, row1)
        out[lo - row0: hi - row0] = bg[lo - a: hi - a]
    return out


def generate_scene(lines: int, samples: int, bands: int, seed: int, rate: float = 0.002,
                   device="cpu"):
    cube = generate_rows(lines, samples, bands, seed, 0, lines, rate, device)
    truth, _ = anomaly_plan(lines, samples, rate, seed)
    return cube, truth


# BASELINE.json configs (C4 orientation: 512 lines x 614 samples)
CONFIGS = {
    "C1": dict(lines=64, samples=64, bands=189, rate=0.002, seed=0x12010001),
    "C2": dict(lines=100, samples=100, bands=189, rate=0.002, seed=0x12010002),
    "C3": dict(lines=100, samples=100, bands=189, rate=0.002, seed=0x12010003),
    "C4": dict(lines=512, samples=614, bands=224, rate=0.001, seed=0x12010004),
    "C5": dict(lines=4096, samples=4096, bands=224, rate=0.001, seed=0x12010005),
}
