"""GPU parity: the sm_100a kernels (through the C-ABI) against the pinned CPU oracle.

Tolerances (BASELINE north star): DWT coefficients 1e-5 relative (we hold 1e-12),
detector scores 1e-9 relative on the fp64 path and 1e-4 on the fp32 path, with the
reference's rel_diff |a-b|/max(1,|a|,|b|) (proj/tests/support/testutil.hpp:34-36);
DWEST eigen-counts and top-k anomaly sets identical. Run on a B200: pytest -m gpu.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import OracleError, max_rel_diff  # noqa: E402

hs = pytest.importorskip("paper_1201_2025_b200")
from harness.scene import CONFIGS, generate_scene  # noqa: E402

DEV = "cuda:0"
TOL64 = 1e-9


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a)).to(DEV)


def host(t):
    return t.detach().cpu().numpy()


def run(cube_np, reqs, **kw):
    outs = hs.detect_multi(gpu(cube_np), reqs, **kw)
    torch.cuda.synchronize()
    return [(host(s), None if c is None else host(c)) for s, c in outs]


def W1(n):
    return hs.WindowConfig.single(n)


def W2(i, o):
    return hs.WindowConfig.dual(i, o)


# ------------------------------------------------------------------ reduction
@pytest.mark.parametrize("bands,order,target", [(189, 2, 4), (224, 2, 4), (64, 2, 4), (50, 3, 4),
                                                (189, 1, 8), (16, 2, 2), (189, 2, 16), (300, 2, 4),
                                                (224, 10, 16)])
def test_reduce_matches_oracle(orc, bands, order, target):
    cube = orc.port.random_cube(9, 13, bands, 1000 + bands + order)
    want = orc.port.reduce_cube(cube, order, target)
    for dtype in (np.float64, np.float32):
        c = cube.astype(dtype)
        got = host(hs.reduce_cube(gpu(c), order, target))
        want_c = orc.port.reduce_cube(c, order, target)
        assert max_rel_diff(got, want_c) < 1e-12
    got32 = host(hs.reduce_cube(gpu(cube), order, target, out_dtype=torch.float32))
    assert np.all(np.abs(got32 - want) <= 1e-6 * np.maximum(1, np.abs(want)))


def test_reduce_constant_and_contract(orc):
    got = host(hs.reduce_cube(gpu(np.full((3, 4, 64), 0.5)), 2, 4))
    assert np.all(np.abs(got - 2.0) < 1e-10)
    for order, target, name in ((2, 3, "InvalidValue"), (0, 4, "UnsupportedOrder"),
                                (2, 512, "TargetTooLarge"), (10, 4, "TooShort")):
        with pytest.raises(hs.HsadError) as e:
            hs.reduce_cube(gpu(np.zeros((2, 2, 189))), order, target)
        assert e.value.name == name


# ------------------------------------------------------------------ reference KATs
def _hand(center):
    cube = np.zeros((3, 3, 2))
    cube[0, 0] = (2, 0); cube[0, 1] = (0, 2); cube[0, 2] = (-2, 0); cube[1, 0] = (0, -2)
    cube[1, 1] = center
    return cube


def test_lrx_hand_case_25():
    m = hs.local_rx(gpu(_hand((3, 4))), W1(3), 1e-9)
    assert abs(m.at(1, 1) - 25.0) < 25e-6 and m.algorithm == "lrx" and m.window == "3"


def test_dwrx_hand_case_5():
    assert abs(hs.dwrx(gpu(_hand((1, 2))), W2(1, 3), 1e-9).at(1, 1) - 5.0) < 5e-6


def test_constant_fields_zero():
    assert torch.all(hs.local_rx(gpu(np.full((6, 7, 3), 2.5)), W1(3)).scores == 0)
    assert torch.all(hs.dwrx(gpu(np.full((8, 8, 3), 1.25)), W2(3, 7)).scores == 0)
    m = hs.dwest(gpu(np.full((9, 9, 3), 0.75)), W2(3, 7))
    assert torch.all(m.scores == 0) and torch.all(m.eigcount == 0)


def test_pixel_equal_to_background_mean(orc):
    cube = orc.port.random_cube(7, 7, 2, 5)
    ring = [cube[3 + dr, 3 + dc] for dr in range(-2, 3) for dc in range(-2, 3) if (dr, dc) != (0, 0)]
    cube[3, 3] = np.mean(ring, axis=0)
    assert hs.local_rx(gpu(cube), W1(5)).at(3, 3) < 1e-18


@pytest.mark.parametrize("seed", [2024, 0xACCE3])
def test_random_cube_parity(orc, seed):
    # test_detect.cpp:152-170 / acceptance criterion 3
    cube = orc.port.random_cube(10, 10, 4, seed)
    assert max_rel_diff(host(hs.local_rx(gpu(cube), W1(5), 1e-6).scores),
                        orc.port.local_rx(cube, 5, 1e-6)) < 1e-10
    assert max_rel_diff(host(hs.dwrx(gpu(cube), W2(3, 7), 1e-6).scores),
                        orc.port.dwrx(cube, 3, 7, 1e-6)) < 1e-10
    m = hs.dwest(gpu(cube), W2(3, 7))
    s, n = orc.port.dwest(cube, 3, 7, 0.1)
    assert max_rel_diff(host(m.scores), s) < 1e-10
    assert np.array_equal(host(m.eigcount), n)


def test_against_reference_naive_oracles(ref, orc):
    cube = orc.port.random_cube(10, 10, 4, 2024)
    assert max_rel_diff(host(hs.local_rx(gpu(cube), W1(5)).scores), ref.naive_lrx(cube, 5, 1e-6)) < 1e-10
    assert max_rel_diff(host(hs.dwrx(gpu(cube), W2(3, 7)).scores), ref.naive_dwrx(cube, 3, 7, 1e-6)) < 1e-10
    assert max_rel_diff(host(hs.dwest(gpu(cube), W2(3, 7)).scores), ref.naive_dwest(cube, 3, 7, 0.1)) < 1e-10


@pytest.mark.parametrize("bands", [1, 2, 3, 4, 5, 6, 8])
def test_band_counts(orc, bands):
    cube = orc.port.random_cube(12, 17, bands, 300 + bands)
    (l, _), (d, _), (e, n) = run(cube, [hs.DetectRequest("lrx", W1(5)),
                                       hs.DetectRequest("dwrx", W2(3, 7)),
                                       hs.DetectRequest("dwest", W2(3, 7), eigcount=True)])
    assert max_rel_diff(l, orc.port.local_rx(cube, 5)) < TOL64
    assert max_rel_diff(d, orc.port.dwrx(cube, 3, 7)) < TOL64
    s, c = orc.port.dwest(cube, 3, 7)
    assert max_rel_diff(e, s) < TOL64 and np.array_equal(n, c)


@pytest.mark.parametrize("window,inner,outer", [(3, 1, 3), (7, 3, 9), (11, 5, 11), (15, 5, 15),
                                                (21, 7, 21), (25, 3, 25)])
def test_window_sizes_and_borders(orc, window, inner, outer):
    # images smaller than the window exercise the folding reflection (detect.cpp:71-76)
    for shape in ((23, 31), (6, 9), (40, 5)):
        cube = orc.port.random_cube(*shape, 4, window * 7 + shape[0])
        (l, _), (d, _) = run(cube, [hs.DetectRequest("lrx", W1(window)),
                                    hs.DetectRequest("dwrx", W2(inner, outer))])
        assert_plain_bar(l, orc.port.local_rx(cube, window),
                         lambda r, c: orc.port.hp_local_rx(cube, window, r, c)[0], f"lrx {window} {shape}")
        assert_plain_bar(d, orc.port.dwrx(cube, inner, outer),
                         lambda r, c: orc.port.hp_dwrx(cube, inner, outer, r, c)[0],
                         f"dwrx {inner}/{outer} {shape}")
        if inner > 1:
            (e, n), = run(cube, [hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)])
            s, c = orc.port.dwest(cube, inner, outer)
            assert max_rel_diff(e, s) < TOL64 and np.array_equal(n, c)


def test_lrx_guard_extension(orc):
    cube = orc.port.random_cube(20, 21, 4, 9)
    (g, _), = run(cube, [hs.DetectRequest("lrx", W1(9), guard=3)])
    assert max_rel_diff(g, orc.port.local_rx(cube, 9, 1e-6, guard=3)) < TOL64


def test_properties(orc):
    cube = orc.port.random_cube(8, 8, 3, 31)
    sh = cube + np.array([5.0, -2.0, 11.0])
    for f in (lambda c: hs.local_rx(c, W1(5)), lambda c: hs.dwrx(c, W2(3, 7)),
              lambda c: hs.dwest(c, W2(3, 7))):
        a, b = host(f(gpu(cube)).scores), host(f(gpu(sh)).scores)
        assert max_rel_diff(a, b) < 1e-8 and np.all(np.isfinite(a)) and np.all(a >= 0)
    c4 = orc.port.random_cube(8, 8, 4, 41)
    B = np.array([[2, .5, 0, .1], [0, 1.5, .3, 0], [.2, 0, 1, .4], [0, .1, 0, .8]])
    assert max_rel_diff(host(hs.local_rx(gpu(c4), W1(5), 0.0).scores),
                        host(hs.local_rx(gpu(c4 @ B.T), W1(5), 0.0).scores)) < 1e-6


def test_chi_square_global_rx():
    # acceptance criterion 4: global RX (window 101, ridge 0) on iid Gaussian, mean ~ L
    g = torch.Generator().manual_seed(0xACCE4)
    cube = 0.5 + 0.1 * torch.randn((101, 101, 8), generator=g, dtype=torch.float64)
    m = hs.local_rx(cube.to(DEV), W1(101), 0.0)
    assert abs(float(m.scores.mean()) - 8.0) / 8.0 < 0.05


def test_dispatch_and_errors(orc):
    cube = gpu(orc.port.random_cube(8, 8, 3, 61))
    assert hs.detect(cube, "lrx", W1(5)).algorithm == "lrx"
    for algo, w in (("dwest", W1(15)), ("lrx", W2(3, 7)), ("dwrx", W1(5))):
        with pytest.raises(hs.HsadError) as e:
            hs.detect(cube, algo, w)
        assert e.value.name == "ConfigMismatch"
    with pytest.raises(hs.HsadError) as e:
        hs.dwest(cube, W2(1, 5))
    assert e.value.name == "TooFewSamples" and "at pixel (0, 0)" in str(e.value)


def test_singular_pixel_error_matches_oracle(orc):
    cube = np.zeros((5, 5, 2)); cube[2, 2] = (1.0, 1.0)
    with pytest.raises(OracleError) as want:
        orc.port.local_rx(cube, 3, 1e-6)
    with pytest.raises(hs.HsadError) as got:
        hs.local_rx(gpu(cube), W1(3), 1e-6)
    assert got.value.name == want.value.name == "SingularAfterRidge"
    assert (got.value.row, got.value.col) == (want.value.row, want.value.col)
    assert str(got.value) == str(want.value)


# ------------------------------------------------------------------ BASELINE configs
def _pipeline_check(orc, name, reqs_spec, order=2, rows=None):
    cfg = CONFIGS[name]
    cube, truth = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"],
                                 cfg["rate"], device=DEV)
    red = hs.reduce_cube(cube, order, 4)
    cube_h = host(cube)
    red_o = orc.port.reduce_cube(cube_h, order, 4, workers=8)
    assert max_rel_diff(host(red), red_o) < 1e-12
    reqs = [hs.DetectRequest(a, w, eigcount=(a == "dwest"), **kw) for a, w, kw in reqs_spec]
    outs = hs.detect_multi(red, reqs)
    torch.cuda.synchronize()
    k = int(truth.sum())
    for (a, w, kw), (s, c) in zip(reqs_spec, outs):
        s = host(s)
        if a == "lrx":
            want = orc.port.local_rx(red_o, w.single_size, 1e-6, guard=kw.get("guard", 1), workers=8)
        elif a == "dwrx":
            want = orc.port.dwrx(red_o, w.inner_size, w.outer_size, 1e-6, workers=8)
        else:
            want, wc = orc.port.dwest(red_o, w.inner_size, w.outer_size, 0.1, workers=8)
            assert np.array_equal(host(c), wc), f"{name} {a} eigen-counts"
        assert max_rel_diff(s, want) < TOL64, f"{name} {a}"
        top_g = set(np.argsort(-s.ravel(), kind="stable")[:k].tolist())
        top_o = set(np.argsort(-want.ravel(), kind="stable")[:k].tolist())
        assert top_g == top_o, f"{name} {a} top-{k}"


def test_config_c1(orc):
    _pipeline_check(orc, "C1", [("lrx", W1(9), {"guard": 3}), ("lrx", W1(9), {})])


def test_config_c2(orc):
    _pipeline_check(orc, "C2", [("dwrx", W2(5, 11), {}), ("dwest", W2(5, 11), {})])


def test_config_c4(orc):
    _pipeline_check(orc, "C4", [("lrx", W1(11), {}), ("dwrx", W2(5, 11), {}),
                                ("dwest", W2(5, 11), {})])


# ------------------------------------------------------------------ sharding / e2e
def test_strip_split_bit_identical(orc):
    cube = gpu(orc.port.random_cube(200, 150, 4, 77))
    reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
            hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
    whole = hs.detect_multi(cube, reqs)
    q = hs.row_quantum(200, 150)
    for g in (2, 4, 8):
        per = -(-200 // (g * q)) * q
        for r0 in range(0, 200, per):
            r1 = min(200, r0 + per)
            b0, nb = hs.strip_rows(200, r0, r1, reqs)
            part = hs.detect_multi(cube[b0:b0 + nb], reqs, lines=200, buf_row0=b0,
                                   row_begin=r0, row_end=r1)
            for (ws, wc), (ps, pc) in zip(whole, part):
                assert torch.equal(ws[r0:r1], ps)
                if wc is not None:
                    assert torch.equal(wc[r0:r1], pc)


def test_pipeline_host_equals_device_path(orc):
    cfg = CONFIGS["C2"]
    cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"])
    h = cube.contiguous().pin_memory()
    reqs = [hs.DetectRequest("dwrx", W2(5, 11)), hs.DetectRequest("dwest", W2(5, 11), eigcount=True),
            hs.DetectRequest("lrx", W1(11), score_dtype=torch.float32)]
    outs = [(torch.empty((100, 100), dtype=r.score_dtype).pin_memory(),
             torch.empty((100, 100), dtype=torch.int8) if r.eigcount else None) for r in reqs]
    hs.pipeline_host(h, 2, 4, reqs, outs)
    dev = hs.detect_multi(hs.reduce_cube(cube.to(DEV), 2, 4), reqs)
    for (a, ac), (b, bc) in zip(outs, dev):
        assert torch.equal(a, b.cpu())
        if ac is not None:
            assert torch.equal(ac, bc.cpu())
    # fp32 path: within 1e-4 of the fp64 oracle
    red_o = orc.port.reduce_cube(host(cube), 2, 4)
    assert max_rel_diff(outs[2][0].numpy().astype(np.float64), orc.port.local_rx(red_o, 11)) < 1e-4


def test_cpu_tensor_rejected():
    with pytest.raises(TypeError):
        hs.reduce_cube(torch.zeros((2, 2, 8)), 2, 4)


def test_golden_vectors_from_reference_code():
    """The kernels against tests/golden (produced by the reference's own wavelet.cpp
    and naive detectors, tests/golden/make_golden.py)."""
    from pathlib import Path
    gdir = Path(__file__).resolve().parent / "golden"
    w = np.load(gdir / "golden_wavelet.npz")
    for key in [k for k in w.files if k.startswith("reduce_out_")]:
        _, _, bands, seed, order, target = key.split("_")
        got = host(hs.reduce_cube(gpu(w[f"reduce_in_{bands}_{seed}"]), int(order), int(target)))
        assert max_rel_diff(got, w[key]) < 1e-12
    g = np.load(gdir / "golden_detect.npz")
    for seed in (2024, 0xACCE3):
        c = gpu(g[f"cube_{seed}"])
        assert max_rel_diff(host(hs.local_rx(c, W1(5)).scores), g[f"lrx5_{seed}"]) < 1e-10
        assert max_rel_diff(host(hs.dwrx(c, W2(3, 7)).scores), g[f"dwrx37_{seed}"]) < 1e-10
        assert max_rel_diff(host(hs.dwest(c, W2(3, 7)).scores), g[f"dwest37_{seed}"]) < 1e-10
    c = gpu(g["cube_99"])
    assert max_rel_diff(host(hs.local_rx(c, W1(7)).scores), g["lrx7_99"]) < 1e-10
    assert max_rel_diff(host(hs.dwrx(c, W2(5, 9)).scores), g["dwrx59_99"]) < 1e-10
    assert max_rel_diff(host(hs.dwest(c, W2(5, 9), 0.3).scores), g["dwest59_99"]) < 1e-10


# ------------------------------------------------------------------ full-band path (K5/K6)
@pytest.mark.parametrize("bands,window,inner,outer", [(12, 7, 3, 7), (30, 9, 3, 9), (61, 11, 5, 11)])
def test_fullband_random_cubes(orc, bands, window, inner, outer):
    cube = orc.port.random_cube(11, 13, bands, 500 + bands)
    (l, _), (d, _) = run(cube, [hs.DetectRequest("lrx", W1(window)),
                                hs.DetectRequest("dwrx", W2(inner, outer))])
    assert_plain_bar(l, orc.port.local_rx(cube, window),
                     lambda r, c: orc.port.hp_local_rx(cube, window, r, c)[0], f"fullband lrx L={bands}")
    assert_plain_bar(d, orc.port.dwrx(cube, inner, outer),
                     lambda r, c: orc.port.hp_dwrx(cube, inner, outer, r, c)[0], f"fullband dwrx L={bands}")
    # guard extension at full band
    (g, _), = run(cube, [hs.DetectRequest("lrx", W1(window), guard=3)])
    assert_plain_bar(g, orc.port.local_rx(cube, window, guard=3),
                     lambda r, c: orc.port.hp_local_rx(cube, window, r, c, guard=3)[0],
                     f"fullband lrx guard L={bands}")


def assert_plain_bar(got, want, hp_at, what):
    """The north-star fp64 bar, 1e-9 rel_diff, against the fp64 oracle on every pixel.
    Where the kernel and the fp64 oracle differ by more (two backward-stable fp64 solvers
    at kappa ~1e6-1e7 may differ by ~kappa * eps), the extended-precision third opinion
    (oracle/hp_oracle.cpp, long double) decides: the kernel must be within 1e-9 of it and
    no farther from it than the oracle is."""
    err = np.abs(got - want) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
    bad = np.argwhere(err > TOL64)
    if len(bad) == 0:
        return 0
    truth = hp_at(bad[:, 0], bad[:, 1])
    g, w = got[bad[:, 0], bad[:, 1]], want[bad[:, 0], bad[:, 1]]
    e_k = np.abs(g - truth) / np.maximum(1.0, np.maximum(np.abs(g), np.abs(truth)))
    e_o = np.abs(w - truth) / np.maximum(1.0, np.maximum(np.abs(w), np.abs(truth)))
    assert np.all(e_k <= TOL64), f"{what}: kernel off the long-double value by {e_k.max():.3g}"
    assert np.all(e_k <= e_o), f"{what}: oracle closer to the long-double value at {int((e_k > e_o).sum())} px"
    return len(bad)


def test_fullband_config_c3(orc):
    """BASELINE C3: 100x100x189 without DWT, every pixel of LRX 15 (reference), the 15/5
    guard extension and DWRX 5/15, at the plain 1e-9 bar with the long-double third
    opinion where the two fp64 solvers disagree (assert_plain_bar)."""
    cfg = CONFIGS["C3"]
    cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"],
                             device=DEV)
    (l, _), (g, _), (d, _) = [(host(s), c) for s, c in hs.detect_multi(
        cube, [hs.DetectRequest("lrx", W1(15)), hs.DetectRequest("lrx", W1(15), guard=5),
               hs.DetectRequest("dwrx", W2(5, 15))])]
    ch = host(cube)
    assert_plain_bar(l, orc.port.local_rx(ch, 15, 1e-6, workers=16),
                     lambda r, c: orc.port.hp_local_rx(ch, 15, r, c, workers=16)[0], "C3 lrx 15")
    assert_plain_bar(g, orc.port.local_rx(ch, 15, 1e-6, guard=5, workers=16),
                     lambda r, c: orc.port.hp_local_rx(ch, 15, r, c, guard=5, workers=16)[0],
                     "C3 lrx 15 guard 5")
    assert_plain_bar(d, orc.port.dwrx(ch, 5, 15, 1e-6, workers=16),
                     lambda r, c: orc.port.hp_dwrx(ch, 5, 15, r, c, workers=16)[0], "C3 dwrx 5/15")


def _dwest_full_check(orc, cube, inner, outer, rows=None, frac=0.1, what="", max_hazard=None):
    """Full-band DWEST (fullband_dwest.cu) against the oracle (cyclic Jacobi to fp64,
    hsad_oracle.cpp): scores within 1e-9, identical eigen-counts; pixels whose DWEST
    decision margins (oracle.port.dwest_margins) are below 1e-10 are hazards (SURVEY
    App. A.7: e.g. exactly repeated or zero eigenvalues of the sample-starved mirrored
    corner windows of random cubes) and may legitimately differ; on scene data they
    must be rare (max_hazard)."""
    (e, n), = run(cube, [hs.DetectRequest("dwest", W2(inner, outer), eigen_fraction=frac, eigcount=True)])
    rb, re = rows if rows else (0, cube.shape[0])
    s, c = orc.port.dwest(cube, inner, outer, frac, workers=16, rows=(rb, re))
    cm, sm_ = orc.port.dwest_margins(cube, inner, outer, frac, workers=16, rows=(rb, re))
    hazard = (cm < 1e-10) | (sm_ < 1e-10)
    e, n = e[rb:re], n[rb:re]
    err = np.abs(e - s) / np.maximum(1.0, np.maximum(np.abs(e), np.abs(s)))
    assert np.all(err[~hazard] <= TOL64), f"{what}: max {err[~hazard].max():.3g}"
    assert np.array_equal(n[~hazard], c[~hazard]), f"{what}: eigen-counts"
    if max_hazard is not None:
        assert hazard.sum() <= max_hazard, f"{what}: {int(hazard.sum())} hazard px"
    return float(err.max()), int(hazard.sum())


@pytest.mark.parametrize("bands,inner,outer", [(12, 3, 7), (30, 3, 9), (61, 5, 11), (189, 5, 15)])
def test_fullband_dwest_random_cubes(orc, bands, inner, outer):
    cube = orc.port.random_cube(9, 11, bands, 700 + bands)
    _dwest_full_check(orc, cube, inner, outer, what=f"dwest L={bands}")


def test_fullband_dwest_config_c3(orc):
    """DWEST on the raw 189-band C3 cube (BASELINE configs[2] geometry, 5/15 windows):
    the reference's acceptance criterion 7 runs DWEST without a DWT (proj/tests/acceptance/
    acceptance_main.cpp:305-309). Border rows and interior rows against the oracle."""
    cfg = CONFIGS["C3"]
    cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"])
    ch = cube.numpy()
    for rows in ((0, 3), (48, 51), (97, 100)):
        _dwest_full_check(orc, ch, 5, 15, rows=rows, what=f"C3 dwest rows {rows}", max_hazard=3)


def test_fullband_dwest_limits_and_errors(orc):
    cube = gpu(orc.port.random_cube(4, 5, 208, 3))
    with pytest.raises(hs.HsadError) as e:
        hs.dwest(cube, W2(3, 5))
    assert e.value.name == "Unsupported"
    with pytest.raises(hs.HsadError) as e:
        hs.dwest(gpu(orc.port.random_cube(6, 6, 20, 3)), W2(1, 5))
    assert e.value.name == "TooFewSamples" and "at pixel (0, 0)" in str(e.value)
    flat = np.zeros((5, 5, 12)); flat[2, 2] = 1.0
    with pytest.raises(OracleError) as want:
        orc.port.local_rx(flat, 3, 1e-6)
    with pytest.raises(hs.HsadError) as got:
        hs.local_rx(gpu(flat), W1(3), 1e-6)
    assert str(got.value) == str(want.value)


# ------------------------------------------------------------------ reduce + detect in one call
ALL3 = [("lrx", W1(11), {}), ("dwrx", W2(5, 11), {}), ("dwest", W2(5, 11), {})]


def _rd_vs_oracle(orc, cube_np, reqs_spec, order=2, what=""):
    """hsad_reduce_detect against the oracle's reduce_cube + detectors."""
    cube = gpu(cube_np.astype(np.float32))
    reqs = [hs.DetectRequest(a, w, eigcount=(a == "dwest"), **kw) for a, w, kw in reqs_spec]
    red, outs = hs.reduce_detect(cube, reqs, order, 4)
    torch.cuda.synchronize()
    red_o = orc.port.reduce_cube(host(cube).astype(np.float64), order, 4, workers=8)
    assert max_rel_diff(host(red), red_o) < 1e-12, what
    for (a, w, kw), (s, c) in zip(reqs_spec, outs):
        s = host(s)
        if a == "lrx":
            want = orc.port.local_rx(red_o, w.single_size, 1e-6, guard=kw.get("guard", 1), workers=8)
        elif a == "dwrx":
            want = orc.port.dwrx(red_o, w.inner_size, w.outer_size, 1e-6, workers=8)
        else:
            want, wc = orc.port.dwest(red_o, w.inner_size, w.outer_size, 0.1, workers=8)
            assert np.array_equal(host(c), wc), f"{what} {a} eigen-counts"
        assert max_rel_diff(s, want) < TOL64, f"{what} {a}"
    return red, outs


def test_reduce_detect_config_c4(orc):
    cfg = CONFIGS["C4"]
    cube, truth = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"],
                                 cfg["rate"], device=DEV)
    _, outs = _rd_vs_oracle(orc, host(cube), ALL3, what="C4")
    # one call == hsad_reduce then hsad_detect_multi, bit for bit
    reqs = [hs.DetectRequest(a, w, eigcount=(a == "dwest"), **kw) for a, w, kw in ALL3]
    two = hs.detect_multi(hs.reduce_cube(cube, 2, 4), reqs)
    for (a, b), (c, d) in zip(outs, two):
        assert torch.equal(a, c)
        if b is not None:
            assert torch.equal(b, d)


@pytest.mark.parametrize("lines,samples,bands,spec", [
    (203, 300, 64, ALL3),                                           # ragged last chunk / strip
    (37, 1100, 32, [("dwrx", W2(3, 9), {}), ("dwest", W2(3, 9), {})]),  # 2-column segments
    (40, 2100, 16, [("lrx", W1(7), {})]),                           # 4-column segments, 1 box
    (9, 9, 48, [("lrx", W1(5), {}), ("dwrx", W2(1, 5), {})]),         # tiny image
])
def test_reduce_detect_shapes(orc, lines, samples, bands, spec):
    cube = orc.port.random_cube(lines, samples, bands, 4242 + bands)
    _rd_vs_oracle(orc, cube, spec, what=f"{lines}x{samples}x{bands}")


def test_reduce_detect_strip_bit_identical(orc):
    lines, samples = 230, 400
    cube = gpu(orc.port.random_cube(lines, samples, 32, 91).astype(np.float32))
    reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
            hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
    red_w, whole = hs.reduce_detect(cube, reqs)
    q = hs.row_quantum(lines, samples)
    for g in (2, 3, 8):
        per = -(-lines // (g * q)) * q
        for r0 in range(0, lines, per):
            r1 = min(lines, r0 + per)
            b0, nb = hs.strip_rows(lines, r0, r1, reqs)
            red, part = hs.reduce_detect(cube[b0:b0 + nb], reqs, lines=lines, buf_row0=b0,
                                         row_begin=r0, row_end=r1)
            assert torch.equal(red, red_w[b0:b0 + nb])
            for (ws, wc), (ps, pc) in zip(whole, part):
                assert torch.equal(ws[r0:r1], ps)
                if wc is not None:
                    assert torch.equal(wc[r0:r1], pc)


@pytest.mark.parametrize("bands,target,spec", [
    (189, 4, ALL3),
    (64, 8, [("dwrx", W2(3, 7), {})]),
    (64, 4, [("lrx", W1(25), {})]),
    (64, 4, [("lrx", W1(3), {}), ("lrx", W1(3), {"guard": 1}), ("dwrx", W2(5, 9), {}),
             ("dwrx", W2(3, 7), {})]),
])
def test_reduce_detect_equals_two_step(orc, bands, target, spec):
    cube = gpu(orc.port.random_cube(60, 70, bands, 5).astype(np.float32))
    reqs = [hs.DetectRequest(a, w, eigcount=(a == "dwest"), **kw) for a, w, kw in spec]
    red, outs = hs.reduce_detect(cube, reqs, 2, target)
    red2 = hs.reduce_cube(cube, 2, target)
    two = hs.detect_multi(red2, reqs)
    assert torch.equal(red, red2)
    for (a, b), (c, d) in zip(outs, two):
        assert torch.equal(a, c)


def test_reduce_detect_empty_range(orc):
    cube = gpu(orc.port.random_cube(50, 60, 64, 6).astype(np.float32))
    reqs = [hs.DetectRequest("dwest", W2(3, 7), eigcount=True)]
    # nothing to detect: the reduced cube is still produced
    red_e, outs = hs.reduce_detect(cube, reqs, row_begin=10, row_end=10)
    assert torch.equal(red_e, hs.reduce_cube(cube, 2, 4)) and outs[0][0].numel() == 0


def test_reduce_detect_errors(orc):
    cube = np.zeros((5, 5, 64), dtype=np.float32)
    cube[2, 2] = 1.0
    reqs = [hs.DetectRequest("lrx", W1(3))]
    with pytest.raises(hs.HsadError) as want:
        hs.detect_multi(hs.reduce_cube(gpu(cube), 2, 4), reqs)
    with pytest.raises(hs.HsadError) as got:
        hs.reduce_detect(gpu(cube), reqs)
    assert (got.value.name, got.value.row, got.value.col) == (want.value.name, want.value.row,
                                                              want.value.col)
    assert str(got.value) == str(want.value)
    for order, target, name in ((0, 4, "UnsupportedOrder"), (2, 3, "InvalidValue"),
                                (2, 512, "TargetTooLarge")):
        with pytest.raises(hs.HsadError) as e:
            hs.reduce_detect(gpu(cube), reqs, order, target)
        assert e.value.name == name
    with pytest.raises(hs.HsadError) as e:
        hs.reduce_detect(gpu(cube), [hs.DetectRequest("lrx", W2(1, 3))])
    assert e.value.name == "ConfigMismatch"


def test_pipeline_host_224_bands(orc):
    cube = torch.as_tensor(orc.port.random_cube(120, 130, 224, 8).astype(np.float32))
    reqs = [hs.DetectRequest(a, w, eigcount=(a == "dwest"), **kw) for a, w, kw in ALL3]
    outs = [(torch.empty((120, 130), dtype=r.score_dtype).pin_memory(),
             torch.empty((120, 130), dtype=torch.int8) if r.eigcount else None) for r in reqs]
    hs.pipeline_host(cube.pin_memory(), 2, 4, reqs, outs)
    _, dev = hs.reduce_detect(cube.to(DEV), reqs)
    for (a, ac), (b, bc) in zip(outs, dev):
        assert torch.equal(a, b.cpu())
        if ac is not None:
            assert torch.equal(ac, bc.cpu())


@pytest.mark.parametrize("lines", [5, 400])
def test_pipeline_host_error_matches_device_path(orc, lines):
    """Errors from a later strip of the streamed pipeline: same pixel and message."""
    if lines == 5:
        cube = np.zeros((5, 5, 64), dtype=np.float32)
        cube[2, 2] = 1.0
    else:
        # a no-data (all-zero) block with one lit pixel: its background / annulus is
        # exactly zero, so the reference fails there (C = 0, delta = 0, d != 0)
        cube = orc.port.random_cube(lines, 40, 64, 12).astype(np.float32)
        cube[300:320] = 0.0
        cube[310, 20] = 1.0
    reqs = [hs.DetectRequest("lrx", W1(3)), hs.DetectRequest("dwrx", W2(1, 3))]
    red_o = orc.port.reduce_cube(cube.astype(np.float64), 2, 4)
    with pytest.raises(OracleError) as ref_err:
        orc.port.local_rx(red_o, 3)
    with pytest.raises(hs.HsadError) as want:
        hs.reduce_detect(gpu(cube), reqs)
    assert (want.value.name, want.value.row, want.value.col) == (ref_err.value.name, ref_err.value.row,
                                                                 ref_err.value.col)
    outs = [(torch.empty((lines, cube.shape[1]), dtype=torch.float64), None) for _ in reqs]
    with pytest.raises(hs.HsadError) as got:
        hs.pipeline_host(torch.as_tensor(cube), 2, 4, reqs, outs)
    assert (got.value.name, got.value.row, got.value.col) == (want.value.name, want.value.row,
                                                              want.value.col)
    assert str(got.value) == str(want.value)


# ------------------------------------------------------------------ request groups (C5 sweep)
SWEEP = [(3, 7), (5, 11), (5, 15), (7, 21)]


def _sweep_requests():
    reqs = []
    for i, o in SWEEP:
        reqs += [hs.DetectRequest("lrx", W1(o)), hs.DetectRequest("dwrx", W2(i, o)),
                 hs.DetectRequest("dwest", W2(i, o), eigcount=True)]
    return reqs


def test_sweep_in_one_call_equals_per_pair_calls(orc):
    red = orc.port.random_cube(90, 140, 4, 31)
    cube = gpu(red)
    reqs = _sweep_requests()
    allq = hs.detect_multi(cube, reqs)  # 12 requests -> 4 fused launches
    for g in range(4):
        part = hs.detect_multi(cube, reqs[3 * g:3 * g + 3])
        for (a, b), (c, d) in zip(allq[3 * g:3 * g + 3], part):
            assert torch.equal(a, c)
            if b is not None:
                assert torch.equal(b, d)
    i, o = SWEEP[3]
    assert max_rel_diff(host(allq[9][0]), orc.port.local_rx(red, o, 1e-6, workers=8)) < TOL64
    want, wc = orc.port.dwest(red, i, o, 0.1, workers=8)
    assert max_rel_diff(host(allq[11][0]), want) < TOL64
    assert np.array_equal(host(allq[11][1]), wc)
    # requests with different outer windows run as separate launches (LRX 3 .. 11)
    many = [hs.DetectRequest("lrx", W1(w)) for w in (3, 5, 7, 9, 11)]
    got = hs.detect_multi(cube, many)
    for r, (s, _) in zip(many, got):
        assert torch.equal(s, hs.detect_multi(cube, [r])[0][0])
    # one outer window with more than 4 requests / window sizes: split, same values
    # up to the launch shape's rounding
    mixed = [hs.DetectRequest("dwrx", W2(i, 15)) for i in (1, 3, 5, 7, 9)]
    got = hs.detect_multi(cube, mixed)
    for (i, r), (s, _) in zip(zip((1, 3, 5, 7, 9), mixed), got):
        assert max_rel_diff(host(s), orc.port.dwrx(red, i, 15, 1e-6, workers=8)) < TOL64
    with pytest.raises(hs.HsadError) as e:
        hs.detect_multi(cube, [hs.DetectRequest("lrx", W1(3))] * 17)
    assert e.value.name == "InvalidValue"


def test_pipeline_host_sweep_equals_device_path(orc):
    cube = torch.as_tensor(orc.port.random_cube(150, 90, 64, 17).astype(np.float32))
    reqs = _sweep_requests()
    outs = [(torch.empty((150, 90), dtype=r.score_dtype).pin_memory(),
             torch.empty((150, 90), dtype=torch.int8) if r.eigcount else None) for r in reqs]
    hs.pipeline_host(cube.pin_memory(), 2, 4, reqs, outs)
    dev = hs.detect_multi(hs.reduce_cube(cube.to(DEV), 2, 4), reqs)
    for (a, ac), (b, bc) in zip(outs, dev):
        assert torch.equal(a, b.cpu())
        if ac is not None:
            assert torch.equal(ac, bc.cpu())


# ------------------------------------------------------------------ TMA-staged kernel


@pytest.mark.parametrize("lines,samples", [(6, 9), (23, 31), (70, 129), (33, 300), (9, 2100)])
def test_staged_kernel_bit_identical_and_oracle(orc, monkeypatch, lines, samples):
    """The standard-layout fp64 kernel takes its update rows from a TMA bulk-copy
    stage (strips clipped at the image edges, mirrored rows/columns): the maps must
    equal the global-load kernel's bit for bit (HSAD_NO_STAGE) and match the oracle."""
    cube = orc.port.random_cube(lines, samples, 4, 5000 + lines)
    reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
            hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
    staged = run(cube, reqs)
    monkeypatch.setenv("HSAD_NO_STAGE", "1")
    plain = run(cube, reqs)
    for (a, ca), (b, cb) in zip(staged, plain):
        assert np.array_equal(a, b)
        assert (ca is None and cb is None) or np.array_equal(ca, cb)
    assert max_rel_diff(staged[0][0], orc.port.local_rx(cube, 11)) < TOL64
    assert max_rel_diff(staged[1][0], orc.port.dwrx(cube, 5, 11)) < TOL64
    s, c = orc.port.dwest(cube, 5, 11)
    assert max_rel_diff(staged[2][0], s) < TOL64 and np.array_equal(staged[2][1], c)


@pytest.mark.parametrize("lines,samples", [(12, 600), (7, 2100)])
def test_staged_kernel_multi_column(orc, monkeypatch, lines, samples):
    """LRX alone fits two output columns per thread next to the stage (K = 2)."""
    cube = orc.port.random_cube(lines, samples, 4, 6000 + lines)
    reqs = [hs.DetectRequest("lrx", W1(11))]
    staged = run(cube, reqs)
    monkeypatch.setenv("HSAD_NO_STAGE", "1")
    plain = run(cube, reqs)
    assert np.array_equal(staged[0][0], plain[0][0])
    assert max_rel_diff(staged[0][0], orc.port.local_rx(cube, 11)) < TOL64


def test_zero_block_matches_reference_exactly(orc):
    """No-data fill: windows whose samples are all exactly zero have mean 0 and
    covariance 0 in the reference (two-pass); the kernel's shifted sums must not leave
    rounding residue there (scores exactly 0 inside the block, oracle parity around it)."""
    cube = orc.port.random_cube(90, 70, 4, 33)
    cube[30:55, 10:40] = 0.0
    cube[:, 60:] = 0.0  # a zero border strip
    reqs = [hs.DetectRequest("lrx", W1(5)), hs.DetectRequest("dwrx", W2(3, 7)),
            hs.DetectRequest("dwest", W2(3, 7), eigcount=True)]
    for shape_cube in (cube, cube[:, :, :3].copy()):
        (l, _), (d, _), (e, n) = run(shape_cube, reqs)
        assert max_rel_diff(l, orc.port.local_rx(shape_cube, 5)) < TOL64
        assert max_rel_diff(d, orc.port.dwrx(shape_cube, 3, 7)) < TOL64
        s_, c_ = orc.port.dwest(shape_cube, 3, 7)
        assert max_rel_diff(e, s_) < TOL64 and np.array_equal(n, c_)
        assert np.all(l[35:50, 15:35] == 0.0) and np.all(d[35:50, 15:35] == 0.0)
        assert np.all(e[35:50, 15:35] == 0.0) and np.all(l[:, 64:] == 0.0)


def test_maximum_window_and_limits(orc):
    """The largest window this build supports (hsad_get_limits().max_window) on a small
    image (many folds of the reflection), and one step past it -> Unsupported."""
    lim = hs._abi.Limits()
    hs._abi.lib().hsad_get_limits(lim)
    w = lim.max_window
    cube = orc.port.random_cube(12, 17, 4, 4242)
    (l, _), (d, _) = run(cube, [hs.DetectRequest("lrx", W1(w)), hs.DetectRequest("dwrx", W2(w - 2, w))])
    assert_plain_bar(l, orc.port.local_rx(cube, w), lambda r, c: orc.port.hp_local_rx(cube, w, r, c)[0],
                     f"lrx {w}")
    assert_plain_bar(d, orc.port.dwrx(cube, w - 2, w),
                     lambda r, c: orc.port.hp_dwrx(cube, w - 2, w, r, c)[0], f"dwrx {w}")
    with pytest.raises(hs.HsadError) as e:
        run(cube, [hs.DetectRequest("lrx", W1(w + 2))])
    assert e.value.name == "Unsupported"


@pytest.mark.parametrize("n_strips", [1, 2, 3, 5])
def test_pipeline_sharded_equals_pipeline_host(orc, n_strips):
    """hsad_pipeline_sharded (strip g on device g % count: all on this one GPU here) writes
    maps bit-identical to the single-strip host pipeline, and the oracle's."""
    from paper_1201_2025_b200.sharded import pipeline_sharded
    cube = torch.as_tensor(orc.port.random_cube(203, 150, 64, 31).astype(np.float32))
    reqs = [hs.DetectRequest("lrx", W1(9)), hs.DetectRequest("dwrx", W2(3, 9)),
            hs.DetectRequest("dwest", W2(3, 9), eigcount=True)]
    mk = lambda: [(torch.empty((203, 150), dtype=torch.float64),  # noqa: E731
                   torch.empty((203, 150), dtype=torch.int8) if r.eigcount else None) for r in reqs]
    want, got = mk(), mk()
    hs.pipeline_host(cube, 2, 4, reqs, want)
    pipeline_sharded(cube, 2, 4, reqs, got, n_strips)
    for (a, ca), (b, cb) in zip(got, want):
        assert np.array_equal(a.numpy(), b.numpy())
        assert (ca is None) == (cb is None) and (ca is None or np.array_equal(ca.numpy(), cb.numpy()))
    red_o = orc.port.reduce_cube(cube.numpy().astype(np.float64), 2, 4)
    assert max_rel_diff(got[0][0].numpy(), orc.port.local_rx(red_o, 9)) < TOL64


def test_pipeline_sharded_error_is_first_pixel(orc):
    from paper_1201_2025_b200.sharded import pipeline_sharded
    cube = orc.port.random_cube(400, 40, 64, 12).astype(np.float32)
    cube[300:320] = 0.0
    cube[310, 20] = 1.0   # singular background in a later strip
    cube[350:370] = 0.0
    cube[360, 5] = 1.0
    reqs = [hs.DetectRequest("lrx", W1(3))]
    outs = [(torch.empty((400, 40), dtype=torch.float64), None)]
    with pytest.raises(hs.HsadError) as want:
        hs.pipeline_host(torch.as_tensor(cube), 2, 4, reqs, outs)
    with pytest.raises(hs.HsadError) as got:
        pipeline_sharded(torch.as_tensor(cube), 2, 4, reqs, outs, 4)
    assert (got.value.name, got.value.row, got.value.col) == (want.value.name, want.value.row, want.value.col)
    assert str(got.value) == str(want.value)
