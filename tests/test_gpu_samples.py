"""dual_window_samples (detect.cpp:150-157) and save_score_map's payload (detect.cpp:291-318)
on the device, against a numpy restatement of gather_box / gather_annulus (detect.cpp:83-117)
and of the fp32 little-endian cast."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _mirror(i, n):
    if n == 1:
        return 0
    period = 2 * (n - 1)
    i = abs(i) % period
    return i if i < n else period - i


def _gather(cube, row, col, inner, outer):
    lines, samples, _ = cube.shape
    ih, oh = inner // 2, outer // 2
    box = [cube[_mirror(row + dr, lines), _mirror(col + dc, samples)]
           for dr in range(-ih, ih + 1) for dc in range(-ih, ih + 1)]
    ann = [cube[_mirror(row + dr, lines), _mirror(col + dc, samples)]
           for dr in range(-oh, oh + 1) for dc in range(-oh, oh + 1)
           if not (abs(dr) <= ih and abs(dc) <= ih)]
    return np.array(box, np.float64), np.array(ann, np.float64)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("inner,outer", [(1, 3), (3, 7), (5, 13), (7, 21)])
def test_dual_window_samples_matches_reference_scan(dtype, inner, outer):
    import paper_1201_2025_b200 as hs
    rng = np.random.default_rng(inner * 100 + outer)
    cube = rng.standard_normal((17, 23, 5)).astype(dtype)
    d = torch.from_numpy(cube).cuda()
    for row, col in [(8, 11), (0, 0), (16, 22), (0, 22), (3, 1), (15, 20)]:
        gi, go = hs.dual_window_samples(d, row, col, hs.WindowConfig.dual(inner, outer))
        wi, wo = _gather(cube, row, col, inner, outer)
        assert gi.shape == wi.shape and go.shape == wo.shape
        assert np.array_equal(gi.cpu().numpy(), wi), (row, col)
        assert np.array_equal(go.cpu().numpy(), wo), (row, col)


def test_dual_window_samples_errors():
    import paper_1201_2025_b200 as hs
    d = torch.zeros((4, 4, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(hs.HsadError) as e:
        hs.dual_window_samples(d, 0, 0, hs.WindowConfig.single(3))
    assert e.value.name == "ConfigMismatch" and "dual_window_samples requires a dual window" in str(e.value)
    with pytest.raises(hs.HsadError):
        hs.dual_window_samples(d, 4, 0, hs.WindowConfig.dual(1, 3))
    # a window larger than the cube reflects repeatedly (mirror_index period), like the reference
    small = torch.arange(2 * 3 * 1, dtype=torch.float64, device="cuda").reshape(2, 3, 1)
    gi, go = hs.dual_window_samples(small, 1, 1, hs.WindowConfig.dual(3, 9))
    wi, wo = _gather(small.cpu().numpy(), 1, 1, 3, 9)
    assert np.array_equal(gi.cpu().numpy(), wi) and np.array_equal(go.cpu().numpy(), wo)


def test_save_score_map_round_trip(tmp_path):
    import paper_1201_2025_b200 as hs
    rng = np.random.default_rng(4)
    cube = torch.from_numpy(rng.standard_normal((12, 9, 4))).cuda()
    m = hs.local_rx(cube, hs.WindowConfig.single(3), 1e-6)
    hs.save_score_map(m, tmp_path / "scores")
    text = (tmp_path / "scores.hdr").read_text()
    assert text == ("ENVI\nsamples = 9\nlines = 12\nbands = 1\nheader offset = 0\n"
                    "file type = ENVI Standard\ndata type = 4\ninterleave = bsq\nbyte order = 0\n")
    back = np.frombuffer((tmp_path / "scores.raw").read_bytes(), dtype="<f4")
    want = m.scores.cpu().numpy().astype(np.float32).ravel()
    assert back.shape == want.shape and np.array_equal(back, want)  # test_detect.cpp:258-260
    # fp32 maps pass through unchanged; large and special values follow the C++ cast
    vals = torch.tensor([0.0, -0.0, 1e-50, 3.5e38, 1e39, 1.0000000596046448], dtype=torch.float64, device="cuda")
    raw = hs.encode_score_map(vals).cpu().numpy().view("<f4")
    with np.errstate(over="ignore"):
        want = vals.cpu().numpy().astype(np.float32)
    assert np.array_equal(raw.view(np.uint32), want.view(np.uint32))
    f32 = torch.tensor([1.5, -2.25], dtype=torch.float32, device="cuda")
    assert np.array_equal(hs.encode_score_map(f32).cpu().numpy().view("<f4"), np.array([1.5, -2.25], np.float32))
