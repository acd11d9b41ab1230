"""Pins the CPU oracle (oracle/hsad_oracle.cpp) before it is trusted as the checker.

Every known-answer and property test the reference keeps for this path
(proj/tests/test_wavelet.cpp, test_stats.cpp, test_detect.cpp, acceptance criterion 3)
is restated here against the oracle, and the oracle is compared with oracle/_ref —
the reference's own wavelet.cpp and naive detectors (tests/support/oracles.cpp)
compiled in place — on the reference's seeded inputs. CPU only.
"""
import math

import numpy as np
import pytest

from oracle import OracleError, max_rel_diff


# ----------------------------------------------------------------- wavelet
def _check_filter_pair(low, high, order, tol):
    n = len(low)
    assert n == 2 * order and len(high) == n
    for k in range(n):
        assert high[k] == (low[n - 1 - k] if k % 2 == 0 else -low[n - 1 - k])
    assert abs(sum(low) - math.sqrt(2)) < tol
    assert abs(sum(high)) < tol
    assert abs(sum(v * v for v in low) - 1.0) < tol
    for k in range(1, n // 2):
        assert abs(sum(low[i] * low[i + 2 * k] for i in range(n - 2 * k))) < tol


def test_haar_and_db4_taps(orc):
    # test_wavelet.cpp:45-65
    low, high = orc.port.daubechies(1)
    r = 1 / math.sqrt(2)
    assert np.allclose(low, [r, r], rtol=1e-15) and np.allclose(high, [r, -r], rtol=1e-15)
    low, _ = orc.port.daubechies(2)
    for got, want in zip(low, [0.4829629131, 0.8365163037, 0.2241438680, -0.1294095226]):
        assert abs(got - want) < 1e-10


def test_admissibility_all_orders(orc):
    # test_wavelet.cpp:20-41, 67-71
    for order in range(1, 11):
        low, high = orc.port.daubechies(order)
        _check_filter_pair(list(low), list(high), order, 1e-12)
    for bad in (0, 11):
        with pytest.raises(OracleError) as e:
            orc.port.daubechies(bad)
        assert e.value.name == "UnsupportedOrder"


def test_taps_match_reference(orc, ref):
    for order in range(1, 11):
        a = orc.port.daubechies(order)
        b = ref.daubechies(order)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_haar_1234(orc):
    # test_wavelet.cpp:73-81
    a, d = orc.port.dwt_level([1, 2, 3, 4], 1)
    r = math.sqrt(2)
    assert np.allclose(a, [3 / r, 7 / r], rtol=1e-14)
    assert np.allclose(d, [-1 / r, -1 / r], rtol=1e-14)


def test_constant_signal_low_branch_only(orc):
    # test_wavelet.cpp:83-89
    a, d = orc.port.dwt_level(np.full(8, 3.75), 2)
    assert np.all(np.abs(a - 3.75 * math.sqrt(2)) < 1e-12) and np.all(np.abs(d) < 1e-12)


def test_dwt_level_contract(orc):
    # test_wavelet.cpp:91-100
    with pytest.raises(OracleError) as e:
        orc.port.dwt_level([1, 2, 3], 2)
    assert e.value.name == "OddLength"
    with pytest.raises(OracleError) as e:
        orc.port.dwt_level([1, 2], 2)
    assert e.value.name == "TooShort"


def test_perfect_reconstruction_and_energy(orc):
    # test_wavelet.cpp:102-115
    for order in (1, 2, 3, 5, 8, 10):
        for n in (32, 64, 128):
            if n < 2 * order:
                continue
            x = orc.port.random_signal(n, 1000 + order * 31 + n)
            a, d = orc.port.dwt_level(x, order)
            assert abs(a @ a + d @ d - x @ x) < 1e-10 * (x @ x)
            assert np.abs(orc.port.idwt_level(a, d, order) - x).max() < 1e-10


def test_dwt_vs_reference_brute_oracle(orc, ref):
    # test_wavelet.cpp:135-147 (brute circular correlation, oracles.cpp:50-72)
    for order in (1, 2, 4, 7, 10):
        for n in (24, 32, 64):
            if n < 2 * order:
                continue
            x = orc.port.random_signal(n, 7000 + order * 13 + n)
            a, d = orc.port.dwt_level(x, order)
            oa, od = ref.brute_dwt(x, order)
            assert np.abs(a - oa).max() < 1e-12 and np.abs(d - od).max() < 1e-12
            ra, rd = ref.dwt_level(x, order)
            assert np.array_equal(a, ra) and np.array_equal(d, rd)


def test_multilevel_gains_and_contract(orc):
    # test_wavelet.cpp:149-194
    assert np.all(np.abs(orc.port.multilevel_approx(np.full(64, 1.5), 2, 4) - 6.0) < 1e-10)
    assert np.all(np.abs(orc.port.multilevel_approx(np.full(189, 2.0), 2, 4) - 16.0) < 1e-9)
    for order in (1, 2, 3):
        for n in (16, 48, 100):
            padded = 1 << (n - 1).bit_length()
            gain = math.sqrt(2) ** (math.log2(padded) - 3)
            got = orc.port.multilevel_approx(np.full(n, 0.8), order, 8)
            assert np.all(np.abs(got - gain * 0.8) < 1e-9)
    for bad, name in ((3, "InvalidValue"), (1, "InvalidValue"), (32, "TargetTooLarge")):
        with pytest.raises(OracleError) as e:
            orc.port.multilevel_approx(np.ones(16), 2, bad)
        assert e.value.name == name


def test_reduce_cube_bitwise_vs_reference(orc, ref):
    # reduce_cube (wavelet.cpp:148-167) of the reference, compiled in place
    cube = orc.port.random_cube(5, 7, 189, 33)
    for order, target in ((2, 4), (3, 4), (1, 8), (10, 16)):
        assert np.array_equal(orc.port.reduce_cube(cube, order, target),
                              ref.reduce_cube(cube, order, target, workers=1))
    # same contract error from both (a 16-sample stage is shorter than 20 taps)
    with pytest.raises(OracleError) as a:
        orc.port.reduce_cube(cube, 10, 4)
    with pytest.raises(OracleError) as b:
        ref.reduce_cube(cube, 10, 4)
    assert a.value.code == b.value.code and str(a.value) == str(b.value)
    # worker-count bit identity (test_wavelet.cpp:228-234)
    c2 = orc.port.random_cube(8, 9, 32, 43)
    assert np.array_equal(orc.port.reduce_cube(c2, 2, 4, 1), orc.port.reduce_cube(c2, 2, 4, 4))


def test_reduce_cube_constant(orc):
    # test_wavelet.cpp:205-210
    r = orc.port.reduce_cube(np.full((3, 4, 64), 0.5), 2, 4)
    assert np.all(np.abs(r - 2.0) < 1e-10)


# ----------------------------------------------------------------- geometry
def test_mirror_index_table(orc):
    # test_detect.cpp:23-33
    for (i, n), want in {(0, 5): 0, (4, 5): 4, (-1, 5): 1, (-2, 5): 2, (5, 5): 3, (6, 5): 2,
                         (9, 5): 1, (-7, 3): 1, (3, 1): 0}.items():
        assert orc.port.mirror_index(i, n) == want


def test_window_validation(orc):
    # test_detect.cpp:35-43
    for mode, a, b in ((0, 2, 0), (0, 1, 0), (1, 5, 5), (1, 5, 6), (1, 4, 9)):
        with pytest.raises(OracleError):
            orc.port.window_validate(mode, a, b)
    orc.port.window_validate(0, 15)
    orc.port.window_validate(1, 5, 13)


# ----------------------------------------------------------------- stats
def test_covariance_vs_reference_brute(orc, ref):
    # test_stats.cpp:89-102
    rng = np.random.default_rng(71)
    s = rng.uniform(-1, 1, (23, 5))
    assert np.abs(orc.port.covariance(s) - ref.brute_covariance(s)).max() < 1e-12
    with pytest.raises(OracleError) as e:
        orc.port.covariance(np.array([[1.0, 2.0]]))
    assert e.value.name == "TooFewSamples"


def test_regularized_inverse(orc):
    # test_stats.cpp:113-159
    inv, d = orc.port.regularized_inverse(np.eye(3), 0.0)
    assert np.abs(inv - np.eye(3)).max() < 1e-14 and d == 0.0
    inv, d = orc.port.regularized_inverse(np.ones((2, 2)), 1e-6)
    assert abs(d - 1e-6) < 1e-18
    assert np.abs((np.ones((2, 2)) + d * np.eye(2)) @ inv - np.eye(2)).max() < 1e-6
    with pytest.raises(OracleError) as e:
        orc.port.regularized_inverse(np.zeros((2, 2)), 1e-6)
    assert e.value.name == "SingularAfterRidge"
    rng = np.random.default_rng(0)
    for dim in (4, 16, 32):
        s = rng.uniform(-1, 1, (3 * dim, dim))
        c = orc.port.covariance(s)
        inv, d = orc.port.regularized_inverse(c, 1e-6)
        assert np.abs((c + d * np.eye(dim)) @ inv - np.eye(dim)).max() < 1e-6


def test_symmetric_eigen_hand_cases_and_reference_jacobi(orc, ref):
    # test_stats.cpp:161-215
    w, v = orc.port.symmetric_eigen(np.diag([1.0, 3.0]))
    assert np.allclose(w, [3, 1]) and v[1, 0] > 0 and v[0, 1] > 0
    w, v = orc.port.symmetric_eigen(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(w, [3, 1], rtol=1e-14)
    r = 1 / math.sqrt(2)
    assert abs(v[0, 0] - r) < 1e-12 and abs(v[1, 0] - r) < 1e-12
    rng = np.random.default_rng(1234)
    for dim in (2, 6, 8, 32):
        a = rng.uniform(-1, 1, (dim, dim)); a = np.tril(a) + np.tril(a, -1).T
        w, v = orc.port.symmetric_eigen(a)
        assert np.abs(v @ np.diag(w) @ v.T - a).max() < 1e-8
        assert np.abs(v.T @ v - np.eye(dim)).max() < 1e-10
        assert np.all(np.diff(w) <= 0)
        rw, rv = ref.jacobi_eigen(a)
        assert np.abs(w - rw).max() < 1e-10
        if dim <= 8:
            assert np.abs(v - rv).max() < 1e-9
    with pytest.raises(OracleError) as e:
        orc.port.symmetric_eigen(np.array([[1.0, 2.0], [3.0, 1.0]]))
    assert e.value.name == "NotSymmetric"


# ----------------------------------------------------------------- detectors
def _hand_cube(center):
    cube = np.zeros((3, 3, 2))
    cube[0, 0] = (2, 0); cube[0, 1] = (0, 2); cube[0, 2] = (-2, 0); cube[1, 0] = (0, -2)
    cube[1, 1] = center
    return cube


def test_lrx_hand_case(orc):
    # test_detect.cpp:76-91 -> 25
    s = orc.port.local_rx(_hand_cube((3, 4)), 3, 1e-9)
    assert abs(s[1, 1] - 25.0) < 25e-6


def test_dwrx_hand_case(orc):
    # test_detect.cpp:112-121 -> 5
    s = orc.port.dwrx(_hand_cube((1, 2)), 1, 3, 1e-9)
    assert abs(s[1, 1] - 5.0) < 5e-6


def test_constant_cubes_score_zero(orc):
    # test_detect.cpp:93-98, 123-135
    assert np.all(orc.port.local_rx(np.full((6, 7, 3), 2.5), 3, 1e-6) == 0.0)
    assert np.all(orc.port.dwrx(np.full((8, 8, 3), 1.25), 3, 7, 1e-6) == 0.0)
    s, n = orc.port.dwest(np.full((9, 9, 3), 0.75), 3, 7, 0.1)
    assert np.all(s == 0.0) and np.all(n == 0)


def test_pixel_equal_to_background_mean(orc):
    # test_detect.cpp:100-110
    cube = orc.port.random_cube(7, 7, 2, 5)
    ring = [cube[3 + dr, 3 + dc] for dr in range(-2, 3) for dc in range(-2, 3) if (dr, dc) != (0, 0)]
    cube[3, 3] = np.mean(ring, axis=0)
    assert orc.port.local_rx(cube, 5, 1e-6)[3, 3] < 1e-18


def test_dwest_selection_rule(orc):
    # test_detect.cpp:137-150: diag(1,-1) keeps the positive branch, |proj| = 3
    w, v = orc.port.symmetric_eigen(np.diag([1.0, -1.0]))
    m = np.array([3.0, 4.0]); proj = 0.0
    for i in range(2):
        if w[i] <= 0.0 or w[i] < 0.1 * w[0]:
            break
        proj += v[:, i] @ m
    assert abs(abs(proj) - 3.0) < 3e-14


@pytest.mark.parametrize("seed", [2024, 0xACCE3])
def test_detectors_match_reference_naive_oracles(orc, ref, seed):
    # test_detect.cpp:152-170 and acceptance criterion 3: < 1e-10
    cube = orc.port.random_cube(10, 10, 4, seed)
    assert max_rel_diff(orc.port.local_rx(cube, 5, 1e-6), ref.naive_lrx(cube, 5, 1e-6)) < 1e-10
    assert max_rel_diff(orc.port.dwrx(cube, 3, 7, 1e-6), ref.naive_dwrx(cube, 3, 7, 1e-6)) < 1e-10
    assert max_rel_diff(orc.port.dwest(cube, 3, 7, 0.1)[0], ref.naive_dwest(cube, 3, 7, 0.1)) < 1e-10


def test_detectors_match_reference_naive_more_shapes(orc, ref):
    cube = orc.port.random_cube(13, 9, 3, 99)
    assert max_rel_diff(orc.port.local_rx(cube, 7, 1e-6), ref.naive_lrx(cube, 7, 1e-6)) < 1e-10
    assert max_rel_diff(orc.port.dwrx(cube, 5, 9, 1e-6), ref.naive_dwrx(cube, 5, 9, 1e-6)) < 1e-10
    assert max_rel_diff(orc.port.dwest(cube, 5, 9, 0.3)[0], ref.naive_dwest(cube, 5, 9, 0.3)) < 1e-10


def test_scores_finite_nonnegative(orc):
    # test_detect.cpp:172-182
    cube = orc.port.random_cube(9, 9, 3, 77)
    for s in (orc.port.local_rx(cube, 5), orc.port.dwrx(cube, 3, 7), orc.port.dwest(cube, 3, 7)[0]):
        assert np.all(np.isfinite(s)) and np.all(s >= 0)


def test_translation_invariance(orc):
    # test_detect.cpp:184-203
    cube = orc.port.random_cube(8, 8, 3, 31)
    sh = cube + np.array([5.0, -2.0, 11.0])
    assert max_rel_diff(orc.port.local_rx(cube, 5), orc.port.local_rx(sh, 5)) < 1e-8
    assert max_rel_diff(orc.port.dwrx(cube, 3, 7), orc.port.dwrx(sh, 3, 7)) < 1e-8
    assert max_rel_diff(orc.port.dwest(cube, 3, 7)[0], orc.port.dwest(sh, 3, 7)[0]) < 1e-8


def test_affine_invariance_ridge_zero(orc):
    # test_detect.cpp:205-223
    cube = orc.port.random_cube(8, 8, 4, 41)
    b = np.array([[2, .5, 0, .1], [0, 1.5, .3, 0], [.2, 0, 1, .4], [0, .1, 0, .8]])
    mapped = cube @ b.T
    assert max_rel_diff(orc.port.local_rx(cube, 5, 0.0), orc.port.local_rx(mapped, 5, 0.0)) < 1e-6


def test_worker_count_bit_identity(orc):
    # test_detect.cpp:225-233
    cube = orc.port.random_cube(10, 11, 3, 53)
    assert np.array_equal(orc.port.local_rx(cube, 5, 1e-6, workers=1),
                          orc.port.local_rx(cube, 5, 1e-6, workers=3))
    assert np.array_equal(orc.port.dwest(cube, 3, 7, workers=1)[0],
                          orc.port.dwest(cube, 3, 7, workers=4)[0])


def test_singular_error_reports_first_pixel(orc):
    # SingularAfterRidge at pixel (r, c) (detect.cpp:127-130): a zero-variance
    # background with a displaced centre cannot be ridged (trace 0)
    cube = np.zeros((5, 5, 2)); cube[2, 2] = (1.0, 1.0)
    with pytest.raises(OracleError) as e:
        orc.port.local_rx(cube, 3, 1e-6, workers=3)
    assert e.value.name == "SingularAfterRidge"
    assert "at pixel (" in str(e.value)
    # neighbours of (2,2) get a rank-1 background that the ridge repairs; (2,2)
    # itself sees an all-zero background (trace 0, nothing to ridge)
    assert (e.value.row, e.value.col) == (2, 2)


def test_dwest_inner_one_too_few_samples(orc):
    with pytest.raises(OracleError) as e:
        orc.port.dwest(orc.port.random_cube(6, 6, 3, 1), 1, 5)
    assert e.value.name == "TooFewSamples" and (e.value.row, e.value.col) == (0, 0)
    assert str(e.value).startswith("TooFewSamples: TooFewSamples: covariance needs at least 2")


def test_lrx_guard_extension_equals_manual_annulus(orc):
    # guard G>1 (BASELINE C1/C3, extension): background = box(W) minus box(G)
    cube = orc.port.random_cube(9, 9, 3, 7)
    got = orc.port.local_rx(cube, 7, 1e-6, guard=3)
    r, c = 4, 4
    bg = np.array([cube[r + dr, c + dc] for dr in range(-3, 4) for dc in range(-3, 4)
                   if not (abs(dr) <= 1 and abs(dc) <= 1)])
    mu = bg.mean(0); C = (bg - mu).T @ (bg - mu) / len(bg)
    C += 1e-6 * np.trace(C) / 3 * np.eye(3)
    d = cube[r, c] - mu
    assert abs(got[r, c] - d @ np.linalg.solve(C, d)) < 1e-9 * max(1, got[r, c])


# ----------------------------------------------------------------- golden fixtures
GOLDEN = __import__("pathlib").Path(__file__).resolve().parent / "golden"


def test_oracle_matches_reference_golden_vectors(orc):
    """tests/golden/*.npz were produced by the reference's own code (make_golden.py);
    this pins the restatement even where oracle/_ref is not built."""
    w = np.load(GOLDEN / "golden_wavelet.npz")
    for order in range(1, 11):
        lo, hi = orc.port.daubechies(order)
        assert np.array_equal(lo, w[f"taps_low_{order}"]) and np.array_equal(hi, w[f"taps_high_{order}"])
    a, d = orc.port.dwt_level([1.0, 2, 3, 4], 1)
    assert np.array_equal(a, w["haar_1234_approx"]) and np.array_equal(d, w["haar_1234_detail"])
    for key in [k for k in w.files if k.startswith("reduce_out_")]:
        _, _, bands, seed, order, target = key.split("_")
        cube = w[f"reduce_in_{bands}_{seed}"]
        assert np.array_equal(orc.port.random_cube(5, 7, int(bands), int(seed)), cube)
        assert np.array_equal(orc.port.reduce_cube(cube, int(order), int(target)), w[key])
    g = np.load(GOLDEN / "golden_detect.npz")
    for seed in (2024, 0xACCE3):
        cube = g[f"cube_{seed}"]
        assert np.array_equal(orc.port.random_cube(10, 10, 4, seed), cube)
        assert max_rel_diff(orc.port.local_rx(cube, 5, 1e-6), g[f"lrx5_{seed}"]) < 1e-10
        assert max_rel_diff(orc.port.dwrx(cube, 3, 7, 1e-6), g[f"dwrx37_{seed}"]) < 1e-10
        assert max_rel_diff(orc.port.dwest(cube, 3, 7, 0.1)[0], g[f"dwest37_{seed}"]) < 1e-10
    cube = g["cube_99"]
    assert max_rel_diff(orc.port.local_rx(cube, 7, 1e-6), g["lrx7_99"]) < 1e-10
    assert max_rel_diff(orc.port.dwrx(cube, 5, 9, 1e-6), g["dwrx59_99"]) < 1e-10
    assert max_rel_diff(orc.port.dwest(cube, 5, 9, 0.3)[0], g["dwest59_99"]) < 1e-10


def test_long_double_third_opinion_pinned(orc):
    """oracle/hp_oracle.cpp (long double) agrees with the fp64 restatement on
    well-conditioned 4-band windows and reproduces the reference's hand case
    (proj/tests/test_detect.cpp:76-91: LRX = 25 with ridge 1e-9)."""
    cube = orc.port.random_cube(12, 13, 4, 2024)
    rows, cols = np.divmod(np.arange(12 * 13), 13)
    for window, guard in ((5, 1), (7, 3)):
        want = orc.port.local_rx(cube, window, 1e-6, guard=guard)
        got, piv = orc.port.hp_local_rx(cube, window, rows, cols, guard=guard)
        assert orc.max_rel_diff(got.reshape(12, 13), want) < 1e-12
        assert np.all(piv >= 1.0)
    want = orc.port.dwrx(cube, 3, 7)
    got, _ = orc.port.hp_dwrx(cube, 3, 7, rows, cols)
    assert orc.max_rel_diff(got.reshape(12, 13), want) < 1e-12
    hand = np.zeros((3, 3, 2))
    hand[0, 0] = (2, 0); hand[0, 1] = (0, 2); hand[0, 2] = (-2, 0); hand[1, 0] = (0, -2)
    hand[1, 1] = (3, 4)
    got, _ = orc.port.hp_local_rx(hand, 3, np.array([1]), np.array([1]), ridge=1e-9)
    assert abs(got[0] - 25.0) < 1e-6
