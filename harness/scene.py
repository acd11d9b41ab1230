"""BASELINE.json's synthetic scene generator (stands in for the paper's AVIRIS cubes).

Background pixel = sum_j alpha_j e_j(b) + N(0, 0.01^2) with alpha ~ Dirichlet(1) over
5 endmembers; each endmember is a sum of 3 Gaussian bumps over the band index,
e(b) = sum_m a_m exp(-((b - c_m)/w_m)^2) with c ~ U[0, L), w ~ U[5, 40], a ~ U[0.1, 1]
(the bump shape of the reference's `peaks` spectra, proj/core/src/synth.cpp:234-247,
taken over the band index). Anomalies: `rate` of the pixels, in clusters of 1-3
pixels, blend a 6th endmember, z = (1 - f) b + f e6 with f ~ U[0.3, 1.0] (the
Eq. 10 sub-pixel model, proj/core/src/synth.cpp:20-27); the truth mask marks the
cluster pixels. fp32 BIP output.

The bytes come from the host generator harness/scene_gen.cpp (xoshiro256++ per row,
the algorithm of proj/core/include/hsad/rng.hpp:13-64), so the GPU arm, the CPU
reference arm and the parity tests consume identical cubes, and any row range (a
rank's strip + halo, a parity sample) is reproduced byte for byte on its own.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
_SO = HERE / "_build" / "libscene.so"
_lib = None


def _scene_lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        lib = C.CDLL(str(_SO))
        D, L, I, U = C.POINTER(C.c_double), C.c_int64, C.c_int, C.c_uint64
        lib.scene_endmembers.argtypes = [I, U, D]
        lib.scene_clusters.restype = L
        lib.scene_clusters.argtypes = [L, L, C.c_double, U, L, C.POINTER(L), C.POINTER(L),
                                       C.POINTER(C.c_int32), D]
        lib.scene_rows.argtypes = [L, L, I, U, L, L, D, D, C.c_double, C.POINTER(C.c_float), I]
        _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def endmembers(bands: int, seed: int) -> np.ndarray:
    e = np.empty((6, bands), np.float64)
    _scene_lib().scene_endmembers(bands, seed, _dp(e))
    return e


def clusters(lines: int, samples: int, rate: float, seed: int):
    lib = _scene_lib()
    n = int(lib.scene_clusters(lines, samples, rate, seed, 0, None, None, None, None))
    rows = np.empty(n, np.int64); cols = np.empty(n, np.int64)
    sizes = np.empty(n, np.int32); fracs = np.empty(n, np.float64)
    P = C.POINTER
    lib.scene_clusters(lines, samples, rate, seed, n, rows.ctypes.data_as(P(C.c_int64)),
                       cols.ctypes.data_as(P(C.c_int64)), sizes.ctypes.data_as(P(C.c_int32)),
                       _dp(fracs))
    return rows, cols, sizes, fracs


_OFFSETS = [(0, 0), (0, 1), (1, 0)]


def anomaly_fill(lines: int, samples: int, rate: float, seed: int, row0: int = 0,
                 row1: int | None = None):
    """Truth mask and blend fraction of rows [row0, row1) (later clusters overwrite)."""
    row1 = lines if row1 is None else row1
    truth = np.zeros((row1 - row0, samples), np.uint8)
    fill = np.zeros((row1 - row0, samples), np.float64)
    rows, cols, sizes, fracs = clusters(lines, samples, rate, seed)
    for r, c, s, f in zip(rows.tolist(), cols.tolist(), sizes.tolist(), fracs.tolist()):
        for dr, dc in _OFFSETS[:s]:
            rr, cc = r + dr, c + dc
            if row0 <= rr < row1 and cc < samples:
                truth[rr - row0, cc] = 1
                fill[rr - row0, cc] = f
    return truth, fill


def anomaly_plan(lines: int, samples: int, rate: float, seed: int):
    truth, fill = anomaly_fill(lines, samples, rate, seed)
    return torch.from_numpy(truth), torch.from_numpy(fill)


def generate_rows_np(lines: int, samples: int, bands: int, seed: int, row0: int, row1: int,
                     rate: float = 0.002, noise: float = 0.01, out: np.ndarray | None = None,
                     threads: int | None = None) -> np.ndarray:
    """Rows [row0, row1) of the scene as an fp32 (rows, samples, bands) numpy array."""
    e = endmembers(bands, seed)
    _, fill = anomaly_fill(lines, samples, rate, seed, row0, row1)
    if out is None:
        out = np.empty((row1 - row0, samples, bands), np.float32)
    assert out.shape == (row1 - row0, samples, bands) and out.dtype == np.float32
    assert out.flags.c_contiguous
    threads = threads or os.cpu_count() or 1
    _scene_lib().scene_rows(lines, samples, bands, seed, row0, row1, _dp(e), _dp(fill), noise,
                            out.ctypes.data_as(C.POINTER(C.c_float)), threads)
    return out


def generate_rows(lines: int, samples: int, bands: int, seed: int, row0: int, row1: int,
                  rate: float = 0.002, device="cpu", noise: float = 0.01,
                  pin: bool = False) -> torch.Tensor:
    """Rows [row0, row1) of the scene as an fp32 (rows, samples, bands) tensor on `device`
    (generated on the host: identical bytes on every device)."""
    host = torch.empty((row1 - row0, samples, bands), dtype=torch.float32,
                       pin_memory=pin and torch.cuda.is_available())
    generate_rows_np(lines, samples, bands, seed, row0, row1, rate, noise, out=host.numpy())
    if torch.device(device).type == "cpu":
        return host
    return host.to(device)


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
