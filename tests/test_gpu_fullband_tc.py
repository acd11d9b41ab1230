"""The tcgen05 (kind::i8, Ozaki split) window Gram of the full-band path, HSAD_FB_TC=1.

stats.cpp:13-29 at L = 189 is the path's one dense contraction (north_star item 4). The
integer Gram is exact, so it is checked (a) entry by entry against an extended-precision
numpy Gram, (b) through LRX / DWRX against the fp64 oracle on well-conditioned cubes at the
plain 1e-9 bar, and (c) on BASELINE C3 (kappa up to 2e6) against the long-double third
opinion: the route must be as close to it as the reference's own fp64 arithmetic is.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_scene
from paper_1201_2025_b200 import _abi

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL64 = 1e-9
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual


def rel(a, b):
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def mirror(i, n):
    if n == 1:
        return 0
    p = 2 * (n - 1)
    i = abs(i) % p
    return i if i < n else p - i


def run(cube, reqs):
    t = cube if isinstance(cube, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(cube)).to(DEV)
    outs = hs.detect_multi(t, reqs)
    torch.cuda.synchronize()
    return [s.cpu().numpy() for s, _ in outs]


@pytest.mark.parametrize("lines,samples,bands,outer,excl",
                         [(24, 70, 189, 15, 1), (30, 90, 189, 15, 5), (20, 40, 60, 9, 3),
                          (9, 11, 150, 21, 0), (16, 33, 127, 7, 1)])
def test_tc_gram_matches_extended_precision(lines, samples, bands, outer, excl):
    """Raw Gram tiles (hi + lo planes) of the shifted samples against numpy long double:
    borders (reflection), walk starts, both column pairs of a guarded window."""
    lib = C.CDLL(str(_abi.LIB_PATH))
    g = torch.Generator(device="cpu").manual_seed(7)
    cube = (torch.rand(lines, samples, bands, generator=g) * 0.8 + 0.1).float()
    cube += 0.3 * torch.rand(lines, samples, 1, generator=g)
    d_cube = cube.to(DEV).contiguous()
    T = (bands + 1 + 7) // 8
    ntile = T * (T + 1) // 2
    gram = torch.full((lines * samples * ntile * 128,), float("nan"), dtype=torch.float64, device=DEV)
    su = torch.zeros(2 * 192, dtype=torch.float64, device=DEV)
    lib.hsad_debug_fb_tc_gram.restype = C.c_int32
    lib.hsad_debug_fb_tc_gram.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                          C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    st = lib.hsad_debug_fb_tc_gram(d_cube.data_ptr(), 4, lines, samples, bands, 0, lines, outer, excl,
                                   gram.data_ptr(), su.data_ptr(), None)
    torch.cuda.synchronize()
    assert st == 0
    planes = gram.cpu().numpy().reshape(lines, samples, ntile, 2, 8, 8)
    shift = su.cpu().numpy()[:192]
    x = cube.numpy().astype(np.float64)
    R, Re = outer // 2, excl // 2
    rng = np.random.default_rng(3)
    pix = [(0, 0), (0, samples - 1), (lines - 1, samples // 2), (lines // 2, min(50, samples - 1)),
           (lines // 2, min(51, samples - 1))] + [(int(rng.integers(lines)), int(rng.integers(samples)))
                                                  for _ in range(4)]
    for r, c in pix:
        ys = [x[mirror(r + dr, lines), mirror(c + dc, samples)] - shift[:bands]
              for dr in range(-R, R + 1) for dc in range(-R, R + 1)
              if not (excl > 0 and abs(dr) <= Re and abs(dc) <= Re)]
        Y = np.array(ys, dtype=np.longdouble)
        G = Y.T @ Y
        S = Y.sum(axis=0)
        full = np.zeros((8 * T, 8 * T), dtype=np.longdouble)
        for ti in range(T):
            for tk in range(ti + 1):
                p = planes[r, c, ti * (ti + 1) // 2 + tk].astype(np.longdouble)
                full[8 * ti:8 * ti + 8, 8 * tk:8 * tk + 8] = p[0] + p[1]
        low = np.tril_indices(bands)
        scale = np.sqrt(np.outer(np.diag(G), np.diag(G)))
        err = float(np.max(np.abs(full[:bands, :bands] - G)[low] / scale[low]))
        assert err < 1e-16, f"Gram ({r},{c}): {err}"  # (hi, lo) is exact; the long-double reference is not
        # row `bands` is the constant-one band: the exact window sums and the sample count
        serr = float(np.max(np.abs(full[bands, :bands] - S) / np.sqrt(np.diag(G))))
        assert serr < 1e-16, f"window sums ({r},{c}): {serr}"
        assert full[bands, bands] == len(ys)


@pytest.mark.parametrize("bands,window,inner,outer", [(12, 7, 3, 7), (30, 9, 3, 9), (61, 11, 5, 11),
                                                      (150, 13, 5, 13)])
def test_tc_route_random_cubes(orc, monkeypatch, bands, window, inner, outer):
    """LRX, the guard extension and DWRX through the tensor-core Gram on random cubes
    (well conditioned): the plain 1e-9 bar against the fp64 oracle, every pixel."""
    monkeypatch.setenv("HSAD_FB_TC", "1")
    cube = orc.port.random_cube(11, 13, bands, 500 + bands)
    l, d, g = run(cube, [hs.DetectRequest("lrx", W1(window)), hs.DetectRequest("dwrx", W2(inner, outer)),
                         hs.DetectRequest("lrx", W1(window), guard=3)])
    assert rel(l, orc.port.local_rx(cube, window)).max() < TOL64
    assert rel(d, orc.port.dwrx(cube, inner, outer)).max() < TOL64
    assert rel(g, orc.port.local_rx(cube, window, guard=3)).max() < TOL64


def test_tc_route_matches_fma_route(orc, monkeypatch):
    """Same maps as the fp64 FMA Gram (1e-9; ~1e-15 away from the reflected borders), fp64 input
    cubes included."""
    cube = orc.port.random_cube(40, 37, 60, 77)
    reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(3, 11))]
    monkeypatch.setenv("HSAD_FB_TC", "0")
    a = run(cube, reqs)
    a64 = run(torch.from_numpy(cube.astype(np.float64)).to(DEV), reqs)
    monkeypatch.setenv("HSAD_FB_TC", "1")
    b = run(cube, reqs)
    b64 = run(torch.from_numpy(cube.astype(np.float64)).to(DEV), reqs)
    for x, y in zip(a + a64, b + b64):
        assert rel(x, y).max() < TOL64, rel(x, y).max()  # interior ~1e-15; mirrored border columns are near-singular


def test_tc_route_config_c3(orc, monkeypatch):
    """BASELINE C3 through the tensor-core Gram, every pixel. At kappa up to 2e6 two fp64
    computations that do not share their rounding differ by ~kappa * eps, so the bar is the
    long-double third opinion: the route's worst and typical distance from it must not
    exceed the fp64 oracle's own, and it stays within 3e-9 of the oracle."""
    monkeypatch.setenv("HSAD_FB_TC", "1")
    cfg = CONFIGS["C3"]
    cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"], device=DEV)
    got, = run(cube, [hs.DetectRequest("lrx", W1(15))])
    ch = cube.cpu().numpy()
    import os
    cores = os.cpu_count() or 1
    want = orc.port.local_rx(ch, 15, 1e-6, workers=cores)
    rows, cols = np.divmod(np.arange(100 * 100), 100)
    truth = np.asarray(orc.port.hp_local_rx(ch, 15, rows, cols, workers=cores)[0]).reshape(100, 100)
    e_k, e_o = rel(got, truth), rel(want, truth)
    assert rel(got, want).max() < 3e-9
    assert e_k.max() <= max(e_o.max(), TOL64) * 1.05, (e_k.max(), e_o.max())
    assert (e_k > TOL64).sum() <= max((e_o > TOL64).sum(), 1) * 1.5
    assert np.median(e_k) < 1e-11


def test_tc_route_row_batches_bit_identical(orc, monkeypatch):
    """The Gram tiles are produced in row batches (<= 4 GB of tiles): forcing batches of 3 and
    of 1 rows must reproduce the one-batch maps bit for bit (same digits, same walks)."""
    monkeypatch.setenv("HSAD_FB_TC", "1")
    cube = orc.port.random_cube(10, 57, 40, 5)
    reqs = [hs.DetectRequest("lrx", W1(7)), hs.DetectRequest("dwrx", W2(3, 7))]
    one = run(cube, reqs)
    for rows in ("3", "1"):
        monkeypatch.setenv("HSAD_TC_BATCH_ROWS", rows)
        for x, y in zip(one, run(cube, reqs)):
            assert np.array_equal(x, y)
