"""The 4-band DWEST eigen route (tridiagonal form, polynomial roots, twisted-factorisation
vectors, Jacobi fallback) at the matrix level: hsad_dwest_pairs runs the fused detectors'
device code on explicit (C_diff, m_diff) pairs, compared with LAPACK (numpy.linalg.eigh)
applying symmetric_eigen's order and sign rule (stats.cpp:64-89) and the DWEST selection
loop (detect.cpp:252-263). Pairs whose selection or sign decision sits inside a 1e-10
margin are hazards of any fp64 solver and are skipped for the score."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _reference(A, m, frac):
    w, V = np.linalg.eigh(A)
    w, V = w[:, ::-1], V[:, :, ::-1]
    k = np.argmax(np.abs(V), axis=1)
    lead = np.take_along_axis(V, k[:, None, :], 1)[:, 0, :]
    V = V * np.where(lead < 0, -1.0, 1.0)[:, None, :]
    sel = (w > 0) & (w >= frac * w[:, :1])
    proj = np.einsum("nij,ni->nj", V, m)
    score = np.abs((proj * sel).sum(1))
    scale = np.maximum(np.abs(A).max((1, 2)), 1e-300)
    # hazards: an eigenvalue within 1e-10 |A| of the cutoff or of zero, a selected eigenvalue
    # within 1e-6 |A| of a neighbour, two components tied for the sign rule
    cut = frac * w[:, :1]
    near_cut = (np.abs(w - cut)[:, 1:] < 1e-10 * scale[:, None]).any(1) | (np.abs(w) < 1e-10 * scale[:, None]).any(1)
    gaps = np.abs(np.diff(w, axis=1)) / scale[:, None]
    near_gap = np.zeros(len(A), bool)
    for j in range(4):
        g = np.minimum(gaps[:, j - 1] if j > 0 else np.inf, gaps[:, j] if j < 3 else np.inf)
        near_gap |= sel[:, j] & (g < 1e-6)
    av = np.sort(np.abs(V), axis=1)
    tie = (sel & ((av[:, -1, :] - av[:, -2, :]) < 1e-9)).any(1)
    return score, sel.sum(1), near_cut | near_gap | tie


def _run(A, m, frac):
    import paper_1201_2025_b200 as hs
    s, c, r = hs.dwest_pairs(torch.from_numpy(A).cuda(), torch.from_numpy(m).cuda(), frac)
    torch.cuda.synchronize()
    return s.cpu().numpy(), c.cpu().numpy().astype(int), r.cpu().numpy().astype(int)


def _sym(rng, n, spectrum):
    """Random orthogonal similarity of the given spectra (n, 4)."""
    Q, _ = np.linalg.qr(rng.standard_normal((n, 4, 4)))
    return np.einsum("nij,nj,nkj->nik", Q, spectrum, Q)


def _check(A, m, frac, what, min_fast=None):
    A = 0.5 * (A + A.transpose(0, 2, 1))
    s, c, r = _run(A, m, frac)
    s0, c0, hazard = _reference(A, m, frac)
    ok = ~hazard
    assert ok.mean() > 0.5, f"{what}: too many hazards ({hazard.mean():.3f})"
    assert np.array_equal(c[ok], c0[ok]), f"{what}: eigen-count mismatch on {np.flatnonzero(ok & (c != c0))[:5]}"
    rel = np.abs(s - s0) / np.maximum(1.0, np.maximum(np.abs(s), np.abs(s0)))
    assert rel[ok].max() <= 1e-9, f"{what}: score rel diff {rel[ok].max():.3e} at {np.argmax(np.where(ok, rel, 0))}"
    assert np.isfinite(s).all(), f"{what}: non-finite score"
    if min_fast is not None:
        assert (r == 0).mean() >= min_fast, f"{what}: only {(r == 0).mean():.3f} on the two-pair route"
    return r


@pytest.mark.parametrize("frac", [1.0, 0.5, 0.1, 1e-3])
def test_random_matrices(frac):
    rng = np.random.default_rng(1201)
    n = 200_000
    A = rng.standard_normal((n, 4, 4))
    m = rng.standard_normal((n, 4))
    _check(A, m, frac, f"gaussian frac {frac}")


def test_detector_like_spectra():
    """C_in - C_ann of the C5 scenes: a few small positive eigenvalues under large negative
    ones (|lambda_1| down to 1e-4 |A|); nearly every pair must settle on the two-pair route."""
    rng = np.random.default_rng(7)
    n = 300_000
    lam = np.stack([10.0 ** rng.uniform(-4, 0, n), np.zeros(n), -10.0 ** rng.uniform(-3, 0, n),
                    -rng.uniform(0.5, 2.0, n)], 1)
    lam[:, 1] = lam[:, 0] * rng.uniform(-0.5, 0.9, n)
    A = _sym(rng, n, lam)
    m = rng.standard_normal((n, 4))
    _check(A, m, 0.1, "detector-like", min_fast=0.95)


def test_scales_and_definiteness():
    rng = np.random.default_rng(3)
    n = 50_000
    base = _sym(rng, n, np.sort(rng.standard_normal((n, 4)), axis=1)[:, ::-1])
    m = rng.standard_normal((n, 4))
    for scale in (1e-200, 1e-30, 1.0, 1e30, 1e150):
        _check(base * scale, m, 0.1, f"scale {scale:g}")
    # negative definite: no positive eigenvalue -> score 0, count 0
    neg = _sym(rng, n, -np.abs(rng.standard_normal((n, 4))) - 0.1)
    s, c, _ = _run(neg, m, 0.1)
    assert (s == 0).all() and (c == 0).all()
    # positive definite with fraction 1e-6: all four selected (general route)
    pos = _sym(rng, n, rng.uniform(0.5, 2.0, (n, 4)))
    _check(pos, m, 1e-6, "positive definite, all selected")


def test_degenerate_matrices():
    """Zero, diagonal, rank-one, repeated-eigenvalue and decoupled matrices: finite scores,
    right counts; scores compared where the selected eigenvectors are determined."""
    rng = np.random.default_rng(5)
    n = 4096
    m = rng.standard_normal((n, 4))
    # zero matrix
    s, c, _ = _run(np.zeros((n, 4, 4)), m, 0.1)
    assert (s == 0).all() and (c == 0).all()
    # diagonal with distinct entries (any order)
    d = rng.permuted(np.tile(np.array([3.0, 1.0, -0.5, -2.0]), (n, 1)), axis=1)
    A = np.zeros((n, 4, 4))
    A[:, range(4), range(4)] = d
    _check(A, m, 0.1, "diagonal")
    # rank one u u^T: one positive eigenvalue, triple zero
    u = rng.standard_normal((n, 4))
    s, c, _ = _run(u[:, :, None] * u[:, None, :], m, 0.1)
    want = np.abs((u * m).sum(1)) / np.linalg.norm(u, axis=1)
    assert (c == 1).all()
    assert np.max(np.abs(s - want) / np.maximum(1, want)) <= 1e-9
    # identity-like: every direction is an eigenvector; count must be 4 and the score finite
    s, c, _ = _run(np.tile(np.eye(4) * 2.5, (n, 1, 1)), m, 0.1)
    assert (c == 4).all() and np.isfinite(s).all()
    # decoupled 2 x 2 blocks (zero off-diagonal couplings in the tridiagonal form)
    B = np.zeros((n, 4, 4))
    B[:, :2, :2] = _sym2(rng, n, 2.0, 0.7)
    B[:, 2:, 2:] = _sym2(rng, n, -0.3, -1.1)
    _check(B, m, 0.1, "2x2 blocks")
    # close pairs inside the selection: gaps 1e-3 .. 1e-7 of |A| (general route below 3e-5)
    for gap in (1e-3, 1e-4, 1e-5, 1e-7):
        lam = np.tile(np.array([1.0, 1.0 - gap, -0.2, -0.9]), (n, 1))
        C = _sym(rng, n, lam)
        s, c, r = _run(C, m, 0.1)
        assert (c == 2).all() and np.isfinite(s).all()
        # any fp64 solver resolves a close pair's vectors to ~eps |A| / gap; compare with
        # LAPACK down to gap 1e-5 at that bar
        s0, c0, hz = _reference(C, m, 0.1)
        ok = ~hz
        if gap >= 1e-5:
            rel = np.abs(s - s0) / np.maximum(1, np.maximum(s, s0))
            assert rel[ok].max() <= max(1e-9, 1e-13 / gap), f"gap {gap}: {rel[ok].max():.3e}"


def _sym2(rng, n, a, b):
    t = rng.uniform(0, np.pi, n)
    c, s = np.cos(t), np.sin(t)
    M = np.empty((n, 2, 2))
    M[:, 0, 0] = c * c * a + s * s * b
    M[:, 1, 1] = s * s * a + c * c * b
    M[:, 0, 1] = M[:, 1, 0] = c * s * (a - b)
    return M


def test_third_eigenvalue_near_cutoff_takes_general_route():
    rng = np.random.default_rng(11)
    n = 20_000
    lam = np.tile(np.array([1.0, 0.5, 0.1 + 1e-8, -0.4]), (n, 1))
    lam[n // 2:, 2] = 0.1 - 1e-8
    A = _sym(rng, n, lam)
    m = rng.standard_normal((n, 4))
    s, c, r = _run(A, m, 0.1)
    assert (r == 1).all()
    assert (c[: n // 2] == 3).all() and (c[n // 2:] == 2).all()


def test_three_selected_eigenvalues_stay_on_the_tridiagonal_route():
    rng = np.random.default_rng(13)
    n = 50_000
    lam = np.stack([rng.uniform(0.8, 1.2, n), rng.uniform(0.4, 0.6, n), rng.uniform(0.15, 0.3, n),
                    -rng.uniform(0.1, 2.0, n)], 1)
    A = _sym(rng, n, lam)
    m = rng.standard_normal((n, 4))
    r = _check(A, m, 0.1, "three selected", min_fast=0.99)
    s, c, _ = _run(0.5 * (A + A.transpose(0, 2, 1)), m, 0.1)
    assert (c == 3).all()
    # four selected: the general route
    lam[:, 3] = rng.uniform(0.125, 0.145, n)  # above every cutoff (<= 0.12)
    B = _sym(rng, n, lam)
    s, c, r = _run(0.5 * (B + B.transpose(0, 2, 1)), m, 0.1)
    assert (c == 4).all() and (r == 1).all()
    _check(B, m, 0.1, "four selected")
