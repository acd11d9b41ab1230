"""CPU pin of the ingest / evaluation oracle against the
reference's own cube.cpp / eval.cpp / pgm.cpp (oracle/_ref/libhsad_ref_io.so), and
the host-side validation of hsad_read_cube / hsad_roc (no GPU needed)."""
import ctypes as C

import numpy as np
import pytest

from oracle import OracleError
from oracle import io_eval as io
from paper_1201_2025_b200 import _abi


@pytest.fixture(scope="module")
def refio():
    r = io.ref_io()
    if r is None:
        pytest.skip("oracle/_ref/libhsad_ref_io.so not built (reference sources absent)")
    return r


def _raw(rng, lines, samples, bands, interleave, code, byte_order):
    dt = {1: np.uint8, 2: np.int16, 4: np.float32, 5: np.float64, 12: np.uint16}[code]
    if code in (4, 5):
        v = rng.normal(0.0, 3.0, size=lines * samples * bands)
    else:
        info = np.iinfo(dt)
        v = rng.integers(info.min, info.max, size=lines * samples * bands, endpoint=True)
    d = np.dtype(dt).newbyteorder(">" if byte_order else "<")
    return v.astype(d).tobytes()


@pytest.mark.parametrize("interleave", ["bsq", "bil", "bip"])
@pytest.mark.parametrize("code", [1, 2, 4, 5, 12])
@pytest.mark.parametrize("byte_order", [0, 1])
def test_read_cube_port_equals_reference(refio, interleave, code, byte_order):
    rng = np.random.default_rng(code * 10 + byte_order)
    lines, samples, bands = 5, 7, 6
    raw = _raw(rng, lines, samples, bands, interleave, code, byte_order)
    a = refio.read_cube(raw, samples, lines, bands, interleave, code, byte_order)
    b = io.read_cube(raw, samples, lines, bands, interleave, code, byte_order)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("args,code,msg", [
    ((0, 3, 2, "bsq", 4, 0), 2, "InvalidValue: samples, lines and bands must all be >= 1"),
    ((3, 3, 2, "bsq", 3, 0), 2, "InvalidValue: unsupported data type code 3"),
    ((3, 3, 2, "bsq", 4, 2), 2, "InvalidValue: byte order must be 0 or 1"),
])
def test_read_cube_validation_errors(refio, args, code, msg):
    raw = bytes(3 * 3 * 2 * 4)
    for fn in (refio.read_cube, io.read_cube):
        with pytest.raises(OracleError) as e:
            fn(raw, *args)
        assert e.value.code == code and str(e.value) == msg


def test_read_cube_size_and_nonfinite(refio):
    raw = np.zeros(3 * 4 * 2, np.float32)
    for fn in (refio.read_cube, io.read_cube):
        with pytest.raises(OracleError) as e:
            fn(raw.tobytes()[:-4], 4, 3, 2, "bsq", 4, 0)
        assert str(e.value) == "SizeMismatch: raw data is 92 bytes, header expects 96"
    # two non-finite values; the first in (row, col, band) order wins
    bsq = raw.reshape(2, 3, 4).copy()
    bsq[1, 0, 1] = np.inf   # band 1, row 0, col 1
    bsq[0, 2, 3] = np.nan   # band 0, row 2, col 3
    for fn in (refio.read_cube, io.read_cube):
        with pytest.raises(OracleError) as e:
            fn(bsq.tobytes(), 4, 3, 2, "bsq", 4, 0)
        assert str(e.value) == "NonFiniteValue: at (row=0, col=1, band=1)"


def _scores_truth(rng, lines, samples, ties=False, rate=0.05):
    s = rng.random((lines, samples))
    if ties:
        s = np.round(s * 20) / 20  # heavy ties
        s[0, 0] = -0.0
        s[0, 1] = 0.0
    t = (rng.random((lines, samples)) < rate).astype(np.uint8)
    t[0, 0], t[-1, -1] = 1, 0
    return s, t


@pytest.mark.parametrize("ties", [False, True])
def test_roc_port_equals_reference(refio, ties):
    rng = np.random.default_rng(7 + ties)
    s, t = _scores_truth(rng, 30, 41, ties)
    f1, t1, a1 = refio.roc_curve(s, t)
    f2, t2, a2, num = io.roc_curve(s, t)
    assert a1 == a2 and np.array_equal(f1, f2) and np.array_equal(t1, t2)
    # the reference's own auc() over the points (trapezoid) agrees to rounding
    area = np.sum(np.diff(f1) * (t1[:-1] + t1[1:]) / 2.0)
    assert abs(area - a1) < 1e-12


def test_roc_degenerate_truth(refio):
    s = np.random.default_rng(0).random((4, 5))
    for t in (np.zeros((4, 5), np.uint8), np.ones((4, 5), np.uint8)):
        with pytest.raises(OracleError) as e:
            refio.roc_curve(s, t)
        assert str(e.value) == "DegenerateTruth: truth mask must contain both classes"
        with pytest.raises(OracleError):
            io.roc_curve(s, t)


def test_threshold_and_pgm_port_equal_reference(refio):
    rng = np.random.default_rng(3)
    s = rng.gamma(2.0, 1.5, size=(37, 29))
    for z in (0.0, 1.5, 3.0):
        ta, ma = refio.adaptive_threshold(s, z)
        tb, mb = io.adaptive_threshold(s, z)
        assert ta == tb and np.array_equal(ma, mb)
    assert refio.render_pgm(s) == io.render_pgm(s)
    c = np.full((3, 4), 2.5)
    assert refio.render_pgm(c) == io.render_pgm(c)  # constant map -> all zero
    half = np.array([[0.0, 0.5 / 255.0, 1.0]])  # exact half-way pixel rounds away from zero
    assert refio.render_pgm(half) == io.render_pgm(half)


def test_read_cube_abi_validates_on_host():
    """hsad_read_cube checks the header and byte count before touching the device."""
    lib = _abi.lib()
    h = _abi.CubeHeader(0, 3, 2, _abi.HSAD_BSQ, 4, 0)
    assert lib.hsad_read_cube(None, 0, C.byref(h), None, 8, None) == _abi.HSAD_E_INVALID_VALUE
    assert lib.hsad_last_error_message() == b"InvalidValue: samples, lines and bands must all be >= 1"
    h = _abi.CubeHeader(4, 3, 2, _abi.HSAD_BSQ, 4, 0)
    assert lib.hsad_read_cube(None, 92, C.byref(h), None, 8, None) == _abi.HSAD_E_SIZE_MISMATCH
    assert lib.hsad_last_error_message() == b"SizeMismatch: raw data is 92 bytes, header expects 96"
    h = _abi.CubeHeader(4, 3, 2, _abi.HSAD_BSQ, 5, 0)
    assert lib.hsad_read_cube(None, 192, C.byref(h), None, 4, None) == _abi.HSAD_E_INVALID_VALUE
