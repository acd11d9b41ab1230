"""GPU parity of the ingest / evaluation kernels (csrc/ingest.cu, csrc/eval.cu)
against the reference's own cube.cpp / eval.cpp / pgm.cpp (oracle/_ref) and the
numpy restatement (oracle/io_eval.py). Integer / byte work: bit-exact."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import io_eval as io  # noqa: E402

hs = pytest.importorskip("paper_1201_2025_b200")
from paper_1201_2025_b200 import evalio  # noqa: E402
from paper_1201_2025_b200.hsad import HsadError  # noqa: E402

DEV = "cuda:0"


def refio_or_port():
    return io.ref_io()


def _raw(rng, lines, samples, bands, code, byte_order):
    dt = {1: np.uint8, 2: np.int16, 4: np.float32, 5: np.float64, 12: np.uint16}[code]
    if code in (4, 5):
        v = rng.normal(0.0, 3.0, size=lines * samples * bands)
    else:
        info = np.iinfo(dt)
        v = rng.integers(info.min, info.max, size=lines * samples * bands, endpoint=True)
    return v.astype(np.dtype(dt).newbyteorder(">" if byte_order else "<")).tobytes()


def _dev(raw: bytes):
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(DEV)


@pytest.mark.parametrize("interleave", ["bsq", "bil", "bip"])
@pytest.mark.parametrize("code", [1, 2, 4, 5, 12])
@pytest.mark.parametrize("byte_order", [0, 1])
@pytest.mark.parametrize("shape", [(5, 7, 6), (33, 70, 189), (3, 1, 40)])
def test_read_cube_bit_exact(interleave, code, byte_order, shape):
    lines, samples, bands = shape
    rng = np.random.default_rng(code * 100 + byte_order * 10 + lines)
    raw = _raw(rng, lines, samples, bands, code, byte_order)
    want = io.read_cube(raw, samples, lines, bands, interleave, code, byte_order)
    r = refio_or_port()
    if r is not None and lines * samples * bands < 100000:
        assert np.array_equal(r.read_cube(raw, samples, lines, bands, interleave, code, byte_order), want)
    hdr = evalio.CubeHeader(samples, lines, bands, interleave, code, byte_order)
    got = evalio.read_cube(_dev(raw), hdr).cpu().numpy()
    assert np.array_equal(got, want)
    if code != 5:  # fp32 holds u8/i16/u16/f32 exactly
        got32 = evalio.read_cube(_dev(raw), hdr, out_dtype=torch.float32).cpu().numpy()
        assert np.array_equal(got32.astype(np.float64), want)


def test_read_cube_errors_match_reference():
    z = np.zeros((2, 3, 4), np.float32)
    z[1, 0, 1] = np.inf
    z[0, 2, 3] = np.nan
    hdr = evalio.CubeHeader(4, 3, 2, "bsq", 4, 0)
    with pytest.raises(HsadError) as e:
        evalio.read_cube(_dev(z.tobytes()), hdr)
    assert str(e.value) == "NonFiniteValue: at (row=0, col=1, band=1)"
    with pytest.raises(HsadError) as e:
        evalio.read_cube(_dev(z.tobytes()[:-4]), hdr)
    assert str(e.value) == "SizeMismatch: raw data is 92 bytes, header expects 96"


def _st(rng, lines, samples, ties, rate=0.05):
    s = rng.random((lines, samples))
    if ties:
        s = np.round(s * 20) / 20
        s[0, 0] = -0.0
        s[0, 1] = 0.0
    t = (rng.random((lines, samples)) < rate).astype(np.uint8)
    t[0, 0], t[-1, -1] = 1, 0
    return s, t


@pytest.mark.parametrize("lines,samples,ties,rate", [(30, 41, False, 0.05), (30, 41, True, 0.05),
                                                     (200, 300, False, 0.002), (64, 64, True, 0.5),
                                                     (1, 2, False, 0.5)])
def test_roc_exact(lines, samples, ties, rate):
    rng = np.random.default_rng(lines + samples + ties)
    s, t = _st(rng, lines, samples, ties, rate)
    far, td, a, num = io.roc_curve(s, t)
    r = refio_or_port()
    if r is not None:
        f1, t1, a1 = r.roc_curve(s, t)
        assert a1 == a and np.array_equal(f1, far) and np.array_equal(t1, td)
    for dtype in (torch.float64, torch.float32):
        sd = torch.as_tensor(s).to(DEV, dtype)
        s_used = sd.double().cpu().numpy()
        far2, td2, a2, num2 = io.roc_curve(s_used, t)
        c = evalio.roc_curve(sd, torch.as_tensor(t).to(DEV))
        assert c.auc_twice_num == num2 and c.auc == a2
        assert np.array_equal(c.far.cpu().numpy(), far2) and np.array_equal(c.td.cpu().numpy(), td2)
        c2 = evalio.roc_curve(sd, torch.as_tensor(t).to(DEV), points=False)
        assert c2.auc == a2


def test_roc_degenerate_and_dimension_errors():
    s = torch.rand(4, 5, dtype=torch.float64, device=DEV)
    with pytest.raises(HsadError) as e:
        evalio.roc_curve(s, torch.zeros(4, 5, dtype=torch.uint8, device=DEV))
    assert str(e.value) == "DegenerateTruth: truth mask must contain both classes"
    with pytest.raises(HsadError) as e:
        evalio.roc_curve(s, torch.zeros(5, 4, dtype=torch.uint8, device=DEV))
    assert e.value.name == "DimensionMismatch"


@pytest.mark.parametrize("n,k,ties", [(1000, 1, False), (1000, 37, False), (5000, 500, True),
                                      (100000, 100, False), (257, 257, True)])
def test_top_k_set(n, k, ties):
    rng = np.random.default_rng(n + k)
    s = rng.random(n)
    if ties:
        s = np.round(s * 10) / 10
    order = np.lexsort((np.arange(n), -s))  # score descending, index ascending
    want = np.sort(order[:k])
    idx, kth = evalio.top_k(torch.as_tensor(s).to(DEV), k)
    assert np.array_equal(idx.cpu().numpy(), want)
    assert kth == s[order[k - 1]]


def test_threshold_and_pgm():
    rng = np.random.default_rng(5)
    s = rng.gamma(2.0, 1.5, size=(97, 131))
    r = refio_or_port()
    for z in (0.0, 2.0, 3.5):
        tau_want, mask_want = (r.adaptive_threshold(s, z) if r is not None else io.adaptive_threshold(s, z))
        res = evalio.adaptive_threshold(torch.as_tensor(s).to(DEV), z)
        # compensated device sums vs the reference's sequential ones: rounding-level tau
        assert abs(res.tau - tau_want) <= 1e-13 * abs(tau_want)
        m = res.mask.cpu().numpy().ravel()
        near = np.abs(s.ravel() - tau_want) <= 1e-12 * abs(tau_want)
        assert np.array_equal(m[~near], mask_want[~near])
    want = r.render_pgm(s) if r is not None else io.render_pgm(s)
    assert evalio.render_pgm(torch.as_tensor(s).to(DEV)) == want
    c = torch.full((3, 4), 2.5, dtype=torch.float64, device=DEV)
    assert evalio.render_pgm(c) == io.render_pgm(np.full((3, 4), 2.5))


@pytest.mark.parametrize("interleave", ["bsq", "bil", "bip"])
@pytest.mark.parametrize("code,byte_order", [(4, 0), (4, 1), (2, 1), (12, 0), (1, 0), (5, 0)])
@pytest.mark.parametrize("lines,samples", [(13, 70), (16, 128)])  # (16, 128): the TMA ring path
def test_reduce_raw_matches_read_then_reduce(orc, interleave, code, byte_order, lines, samples):
    """hsad_reduce_raw == reduce_cube(read_cube(raw)) of the oracle (DWT bar 1e-5; we hold
    1e-10 relative), for every interleave / type / byte order."""
    bands = 189
    rng = np.random.default_rng(code * 7 + byte_order + len(interleave))
    raw = _raw(rng, lines, samples, bands, code, byte_order)
    cube = io.read_cube(raw, samples, lines, bands, interleave, code, byte_order)
    want = orc.port.reduce_cube(cube, 2, 4)
    hdr = evalio.CubeHeader(samples, lines, bands, interleave, code, byte_order)
    got = evalio.reduce_raw(_dev(raw), hdr, 2, 4).cpu().numpy()
    assert orc.max_rel_diff(got, want) < 1e-10  # summation order; int16-scale data cancels


def test_reduce_raw_errors():
    z = np.zeros((64, 3, 4), np.float32)  # BSQ: 64 bands of 3 x 4
    z[10, 2, 1] = np.nan
    hdr = evalio.CubeHeader(4, 3, 64, "bsq", 4, 0)
    with pytest.raises(HsadError) as e:
        evalio.reduce_raw(_dev(z.tobytes()), hdr, 2, 4)
    assert str(e.value) == "NonFiniteValue: at (row=2, col=1, band=10)"
    with pytest.raises(HsadError) as e:
        evalio.reduce_raw(_dev(z.tobytes()), hdr, 11, 4)
    assert e.value.name == "UnsupportedOrder"
    with pytest.raises(HsadError) as e:
        evalio.reduce_raw(_dev(z.tobytes()[:-8]), hdr, 2, 4)
    assert e.value.name == "SizeMismatch"


def test_reduce_raw_large_aligned_nonfinite():
    """A wider aligned BSQ cube: the first non-finite element in (row, col, band) order."""
    rng = np.random.default_rng(77)
    cube = rng.normal(0, 2, size=(224, 16, 256)).astype(np.float32)  # BSQ bands x lines x samples
    hdr = evalio.CubeHeader(256, 16, 224, "bsq", 4, 0)
    cube[100, 7, 200] = np.inf
    cube[150, 3, 9] = np.nan
    with pytest.raises(HsadError) as e:
        evalio.reduce_raw(_dev(cube.tobytes()), hdr, 2, 4)
    assert str(e.value) == "NonFiniteValue: at (row=3, col=9, band=150)"


@pytest.mark.parametrize("interleave,code,byte_order", [("bsq", 4, 0), ("bil", 2, 1), ("bsq", 12, 1)])
def test_pipeline_raw_equals_device_path_and_oracle(orc, interleave, code, byte_order):
    """Host raw ENVI bytes -> hsad_pipeline_raw (streamed strips) == reduce_raw + detect_multi
    on the device (bit for bit) and the oracle's read -> reduce -> detect (1e-9)."""
    lines, samples, bands = 700, 97, 64  # 17 MB: three >= 8 MB strips
    rng = np.random.default_rng(lines + code)
    raw = _raw(rng, lines, samples, bands, code, byte_order)
    hdr = evalio.CubeHeader(samples, lines, bands, interleave, code, byte_order)
    reqs = [hs.DetectRequest("lrx", hs.WindowConfig.single(7)),
            hs.DetectRequest("dwrx", hs.WindowConfig.dual(3, 9)),
            hs.DetectRequest("dwest", hs.WindowConfig.dual(3, 9), eigcount=True)]
    outs = [(torch.empty((lines, samples), dtype=torch.float64),
             torch.empty((lines, samples), dtype=torch.int8) if r.eigcount else None) for r in reqs]
    evalio.pipeline_raw(np.frombuffer(raw, np.uint8).copy(), hdr, 2, 4, reqs, outs)
    red = evalio.reduce_raw(_dev(raw), hdr, 2, 4)
    dev = hs.detect_multi(red, reqs)
    for (a, ca), (b, cb) in zip(outs, dev):
        assert np.array_equal(a.numpy(), b.cpu().numpy())
        assert (ca is None) == (cb is None) and (ca is None or np.array_equal(ca.numpy(), cb.cpu().numpy()))
    cube = io.read_cube(raw, samples, lines, bands, interleave, code, byte_order)
    red_o = orc.port.reduce_cube(cube, 2, 4)
    assert orc.max_rel_diff(outs[0][0].numpy(), orc.port.local_rx(red_o, 7)) < 1e-9
    assert orc.max_rel_diff(outs[1][0].numpy(), orc.port.dwrx(red_o, 3, 9)) < 1e-9
    s_, c_ = orc.port.dwest(red_o, 3, 9)
    assert orc.max_rel_diff(outs[2][0].numpy(), s_) < 1e-9 and np.array_equal(outs[2][1].numpy(), c_)


def test_pipeline_raw_nonfinite_first():
    z = np.zeros((64, 40, 30), np.float32)  # BSQ
    z[:, :, :] = np.random.default_rng(3).random((64, 40, 30)).astype(np.float32)
    z[5, 33, 7] = np.nan
    hdr = evalio.CubeHeader(30, 40, 64, "bsq", 4, 0)
    outs = [(torch.empty((40, 30), dtype=torch.float64), None)]
    with pytest.raises(HsadError) as e:
        evalio.pipeline_raw(np.frombuffer(z.tobytes(), np.uint8).copy(), hdr, 2, 4,
                            [hs.DetectRequest("lrx", hs.WindowConfig.single(5))], outs)
    assert str(e.value) == "NonFiniteValue: at (row=33, col=7, band=5)"
