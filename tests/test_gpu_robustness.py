"""GPU edge cases: misaligned strips into the TMA reduction, failure ordering inside a
fused launch, and the fp32 score path on the BASELINE configs.

* cp.async.bulk needs a 16-byte aligned source; row strips of an odd-samples x
  odd-bands fp32 cube (bands = 189 is the paper's count) start 4 or 8 bytes off.
* A fused group of requests must report what the equivalent sequential hsad::detect
  calls report: the first failing request (in request order), at its first failing
  pixel in row-major order (detect.cpp:127-130, parallel.hpp:17-40).
* The fp32 path (score_bytes = 4) stores fp32 maps of the same fp64 arithmetic:
  within 1e-4 (rel_diff, proj/tests/support/testutil.hpp:34-36) of the fp64 oracle,
  with identical top-k sets and DWEST eigen-counts (BASELINE north star).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import OracleError, max_rel_diff  # noqa: E402

hs = pytest.importorskip("paper_1201_2025_b200")
from harness.scene import CONFIGS, generate_scene  # noqa: E402

DEV = "cuda:0"


def W1(n):
    return hs.WindowConfig.single(n)


def W2(i, o):
    return hs.WindowConfig.dual(i, o)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_reduce_misaligned_row_views(orc, dtype):
    cube = orc.port.random_cube(40, 101, 189, 77).astype(dtype)
    g = torch.as_tensor(cube).to(DEV)
    whole = hs.reduce_cube(g, 2, 4)
    for r in (1, 3, 7):
        view = g[r:]
        assert view.data_ptr() % 16 != 0
        part = hs.reduce_cube(view, 2, 4)
        assert torch.equal(part, whole[r:])  # leading pixels through the lane-split kernel
        assert max_rel_diff(part.cpu().numpy(), orc.port.reduce_cube(cube[r:], 2, 4)) < 1e-12


def test_pipeline_host_odd_samples_odd_bands_many_strips(orc):
    # 1000 x 101 x 189 fp32 = 76 MB: several row strips, each starting off 16-byte alignment
    cube = torch.as_tensor(orc.port.random_cube(1000, 101, 189, 78).astype(np.float32))
    h = cube.pin_memory()
    reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
    outs = [(torch.empty((1000, 101), dtype=torch.float64).pin_memory(),
             torch.empty((1000, 101), dtype=torch.int8) if r.eigcount else None) for r in reqs]
    hs.pipeline_host(h, 2, 4, reqs, outs)
    dev = hs.detect_multi(hs.reduce_cube(cube.to(DEV), 2, 4), reqs)
    for (a, ac), (b, bc) in zip(outs, dev):
        assert torch.equal(a, b.cpu())
        if ac is not None:
            assert torch.equal(ac, bc.cpu())


def _two_failure_cube(orc):
    """LRX 3 (ridge 0) first fails at (5, 5); DWRX 1/5 (ridge 0) first fails later."""
    cube = orc.port.random_cube(20, 20, 4, 79)
    cube[4:7, 4:7] = 0.25          # constant 3x3 background around (5, 5) ...
    cube[5, 5] = (1.0, 0.0, 0.5, 0.0)  # ... with a different centre
    cube[10:15, 10:15] = 0.75      # constant 5x5 annulus around (12, 12) ...
    cube[12, 12] = (0.0, 1.0, 0.0, 0.5)
    return cube


def test_fused_group_reports_first_failing_request(orc):
    cube = _two_failure_cube(orc)
    with pytest.raises(OracleError) as e_dwrx:
        orc.port.dwrx(cube, 1, 5, 0.0)
    with pytest.raises(OracleError) as e_lrx:
        orc.port.local_rx(cube, 3, 0.0)
    p_dwrx = (e_dwrx.value.row, e_dwrx.value.col)
    p_lrx = (e_lrx.value.row, e_lrx.value.col)
    assert p_lrx < p_dwrx  # the later request fails at the earlier pixel
    g = torch.as_tensor(cube).to(DEV)
    # different outer windows: two launches, the first group's failure wins
    reqs = [hs.DetectRequest("dwrx", W2(1, 5), ridge=0.0), hs.DetectRequest("lrx", W1(3), ridge=0.0)]
    with pytest.raises(hs.HsadError) as got:
        hs.detect_multi(g, reqs)
    assert (got.value.row, got.value.col) == p_dwrx
    assert str(got.value) == str(e_dwrx.value)
    # reversed order: LRX is the first request, so its pixel is reported
    with pytest.raises(hs.HsadError) as got2:
        hs.detect_multi(g, reqs[::-1])
    assert (got2.value.row, got2.value.col) == p_lrx
    assert str(got2.value) == str(e_lrx.value)


def _same_window_cube():
    """Integer-valued 24 x 24 x 4 cube (exact sums): LRX 5 (ridge 0) first fails at (4, 4),
    DWRX 3/5 (ridge 0) first fails later, at (16, 16).

    Around (4, 4) the 5x5 box lies in the plane a + t e1 + s e2 (rank-2 background:
    LRX singular, centre off the background mean), while the inner 3x3 mean equals the
    annulus mean exactly (DWRX scores 0 without a solve). Around (16, 16) the annulus
    is constant and the centre differs (DWRX singular)."""
    rng = np.random.default_rng(81)
    cube = rng.integers(0, 8, (24, 24, 4)).astype(np.float64)
    a = np.array([2.0, 2.0, 2.0, 2.0])
    e1 = np.array([1.0, 0, 0, 0]); e2 = np.array([0, 1.0, 0, 0])
    t_ann = iter([1, -1] * 8)
    t_in = iter([1, -1, 1, -1, 1, -1, 1, -1])
    for dr in range(-2, 3):
        for dc in range(-2, 3):
            if max(abs(dr), abs(dc)) == 2:
                cube[4 + dr, 4 + dc] = a + next(t_ann) * e1
            elif (dr, dc) != (0, 0):
                cube[4 + dr, 4 + dc] = a + next(t_in) * e1
    cube[3, 3] += e2            # one ring pixel off the line ...
    cube[4, 4] = a - e2         # ... and the centre opposite: inner mean == annulus mean
    cube[14:19, 14:19] = 5.0
    cube[16, 16] = (1.0, 3.0, 5.0, 7.0)
    return cube


def test_fused_group_same_window_failure_order(orc):
    """LRX and DWRX sharing the outer window run in ONE fused launch; the failure word
    carries the request position, so the first failing request wins over a lower pixel."""
    cube = _same_window_cube()
    want = {}
    for name, fn in (("dwrx", lambda: orc.port.dwrx(cube, 3, 5, 0.0)),
                     ("lrx", lambda: orc.port.local_rx(cube, 5, 0.0))):
        with pytest.raises(OracleError) as e:
            fn()
        want[name] = e.value
    assert (want["lrx"].row, want["lrx"].col) == (4, 4)
    assert (want["dwrx"].row, want["dwrx"].col) == (16, 16)
    g = torch.as_tensor(cube).to(DEV)
    reqs = [hs.DetectRequest("dwrx", W2(3, 5), ridge=0.0), hs.DetectRequest("lrx", W1(5), ridge=0.0)]
    with pytest.raises(hs.HsadError) as got:
        hs.detect_multi(g, reqs)
    assert str(got.value) == str(want["dwrx"])
    with pytest.raises(hs.HsadError) as got2:
        hs.detect_multi(g, reqs[::-1])
    assert str(got2.value) == str(want["lrx"])
    # asynchronous status word: same ordering, decoded by hsad_decode_status
    import ctypes as C
    st = torch.full((1,), -1, dtype=torch.int64, device=DEV)
    hs.detect_multi(g, reqs, status=st)
    torch.cuda.synchronize()
    word = int(st.item()) & (2**64 - 1)
    assert word >> 56 == 0  # request 0 (DWRX)
    e = hs._abi.PixelError()
    assert hs._abi.lib().hsad_decode_status(word, 24, C.byref(e)) == 13
    assert (e.row, e.col) == (16, 16)


@pytest.mark.parametrize("name,spec", [
    ("C1", [("lrx", (9,), {"guard": 3}), ("lrx", (9,), {})]),
    ("C2", [("dwrx", (5, 11), {}), ("dwest", (5, 11), {})]),
    ("C4", [("lrx", (11,), {}), ("dwrx", (5, 11), {}), ("dwest", (5, 11), {})]),
])
def test_fp32_path_on_configs(orc, name, spec):
    cfg = CONFIGS[name]
    cube, truth = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"],
                                 cfg["rate"], device=DEV)
    red = hs.reduce_cube(cube, 2, 4)
    red_o = orc.port.reduce_cube(cube.cpu().numpy(), 2, 4, workers=8)
    reqs = []
    for a, w, kw in spec:
        win = W1(*w) if a == "lrx" else W2(*w)
        reqs.append(hs.DetectRequest(a, win, eigcount=(a == "dwest"), score_dtype=torch.float32, **kw))
    outs = hs.detect_multi(red, reqs)
    torch.cuda.synchronize()
    k = int(truth.sum())
    for (a, w, kw), (s, c) in zip(spec, outs):
        assert s.dtype == torch.float32
        s = s.cpu().numpy().astype(np.float64)
        if a == "lrx":
            want = orc.port.local_rx(red_o, w[0], 1e-6, guard=kw.get("guard", 1), workers=8)
        elif a == "dwrx":
            want = orc.port.dwrx(red_o, w[0], w[1], 1e-6, workers=8)
        else:
            want, wc = orc.port.dwest(red_o, w[0], w[1], 0.1, workers=8)
            assert np.array_equal(c.cpu().numpy(), wc), f"{name} {a} eigen-counts"
        assert max_rel_diff(s, want) < 1e-4, f"{name} {a}"
        top_g = set(np.argsort(-s.ravel(), kind="stable")[:k].tolist())
        top_o = set(np.argsort(-want.ravel(), kind="stable")[:k].tolist())
        assert top_g == top_o, f"{name} {a} top-{k}"


def test_forked_groups_equal_sequential_groups(orc, monkeypatch):
    """An asynchronous multi-group call runs groups 1.. on side streams forked from the
    caller's stream and joined back into it: the maps must equal the sequential launch bit for
    bit, and work queued on the caller's stream right after the call must see every map
    (hsad_detect_multi and hsad_reduce_detect, on a non-default stream)."""
    cube = torch.as_tensor(orc.port.random_cube(150, 260, 64, 11)).float().to(DEV)
    W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
    reqs = []
    for inner, outer in ((3, 7), (5, 11), (5, 15), (7, 21)):
        reqs += [hs.DetectRequest("lrx", W1(outer)), hs.DetectRequest("dwrx", W2(inner, outer)),
                 hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)]
    red = hs.reduce_cube(cube, 2, 4)
    st = torch.full((1,), -1, dtype=torch.int64, device=DEV)

    def sums(fn):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            outs = fn()
            # consumers on the caller's stream, queued right behind the call
            tot = [o[0].sum() for o in outs] + [o[1].double().sum() for o in outs if o[1] is not None]
        side.synchronize()
        return outs, [float(t) for t in tot]

    monkeypatch.setenv("HSAD_NO_FORK", "1")
    seq, seq_sums = sums(lambda: hs.detect_multi(red, reqs, status=st))
    monkeypatch.delenv("HSAD_NO_FORK")
    for _ in range(3):
        frk, frk_sums = sums(lambda: hs.detect_multi(red, reqs, status=st))
        assert frk_sums == seq_sums
        for (a, ac), (b, bc) in zip(seq, frk):
            assert torch.equal(a, b) and (ac is None or torch.equal(ac, bc))
    assert int(st.item()) == -1
    # hsad_reduce_detect: groups 1.. start right after the reduction, next to group 0
    rf, fo = hs.reduce_detect(cube, reqs, 2, 4, status=st)
    torch.cuda.synchronize()
    assert torch.equal(rf, red)
    for (a, ac), (b, bc) in zip(seq, fo):
        assert torch.equal(a, b) and (ac is None or torch.equal(ac, bc))
