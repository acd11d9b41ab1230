"""Checks tc_gram_kernel (tcgen05 kind::i8 window Gram) against numpy on a few pixels.

python scripts/probe_tc_gram.py [lines samples bands outer excl]
Env HSAD_TC_LBO / HSAD_TC_SBO / HSAD_TC_SEG reach the launcher (descriptor strides, walk length).
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1201_2025_b200 import _abi

lib = C.CDLL(str(_abi.LIB_PATH))
args = [int(a) for a in sys.argv[1:]]
lines, samples, bands, outer, excl = (args + [24, 70, 189, 15, 1][len(args):])[:5]
g = torch.Generator(device="cpu").manual_seed(7)
cube = (torch.rand(lines, samples, bands, generator=g) * 0.8 + 0.1).float()
cube += 0.3 * torch.rand(lines, samples, 1, generator=g)
d_cube = cube.cuda().contiguous()
mp = (bands + 1 + 7) // 8 * 8
T = mp // 8
ntile = T * (T + 1) // 2
r0, r1 = 0, lines
gram = torch.full(((r1 - r0) * samples * ntile * 128,), float("nan"), dtype=torch.float64, device="cuda")
su = torch.zeros(2 * 192, dtype=torch.float64, device="cuda")
lib.hsad_debug_fb_tc_gram.restype = C.c_int32
lib.hsad_debug_fb_tc_gram.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                                      C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
st = lib.hsad_debug_fb_tc_gram(d_cube.data_ptr(), 4, lines, samples, bands, r0, r1, outer, excl,
                               gram.data_ptr(), su.data_ptr(), None)
torch.cuda.synchronize()
print("status", st, flush=True)
gram = gram.cpu().numpy().reshape(r1 - r0, samples, ntile, 2, 8, 8).sum(axis=3)
su = su.cpu().numpy()
shift, unit = su[:192], su[192:]
print("shift[:4]", shift[:4], "unit[:4]", unit[:4], "log2", np.log2(unit[:4]))
x = cube.numpy().astype(np.float64)


def mirror(i, n):
    if n == 1:
        return 0
    p = 2 * (n - 1)
    i = abs(i) % p
    return i if i < n else p - i


def ref_gram(r, c):
    R, Re = outer // 2, excl // 2
    ys = []
    for dr in range(-R, R + 1):
        for dc in range(-R, R + 1):
            if excl > 0 and abs(dr) <= Re and abs(dc) <= Re:
                continue
            ys.append(x[mirror(r + dr, lines), mirror(c + dc, samples)] - shift[:bands])
    Y = np.array(ys, dtype=np.longdouble)
    return np.asarray(Y.T @ Y, dtype=np.float64), len(ys)


worst = 0.0
rng = np.random.default_rng(3)
pix = [(0, 0), (0, 1), (0, samples - 1), (lines - 1, samples // 2), (lines // 2, min(49, samples - 1)),
       (lines // 2, min(50, samples - 1)), (lines // 2, min(51, samples - 1))] + [(int(rng.integers(lines)), int(rng.integers(samples))) for _ in range(6)]
for (r, c) in pix:
    G, n = ref_gram(r, c)
    full = np.full((mp, mp), np.nan)
    for ti in range(T):
        for tk in range(ti + 1):
            full[8 * ti:8 * ti + 8, 8 * tk:8 * tk + 8] = gram[r - r0, c, ti * (ti + 1) // 2 + tk]
    low = np.tril_indices(bands)
    got, want = full[:bands, :bands][low], G[low]
    scale = np.sqrt(np.outer(np.diag(G), np.diag(G)))[low]
    err = np.nanmax(np.abs(got - want) / scale) if not np.isnan(got).any() else float("nan")
    nan = int(np.isnan(got).sum())
    worst = max(worst, err if err == err else 1e9)
    pad = full[bands:, :bands]
    print(f"px ({r},{c}) N={n} max |dG|/sqrt(GiiGjj) = {err:.3e} nan={nan} pad max={np.nanmax(np.abs(pad)):.1e} "
          f"G00 got {full[0, 0]:.12g} want {G[0, 0]:.12g}; G[b-1,3] got {full[bands - 1, 3]:.12g} want {G[bands - 1, 3]:.12g}",
          flush=True)
print("worst", worst)
