"""The C-ABI library loads and exports every symbol include/hsad_gpu.h declares;
host-only entry points behave like the reference (no GPU needed)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1201_2025_b200 import _abi

ROOT = Path(__file__).resolve().parents[1]


def test_header_symbols_exported():
    header = (ROOT / "include" / "hsad_gpu.h").read_text()
    declared = set(re.findall(r"\b(hsad_[a-z_]+)\s*\(", header))
    assert declared == set(_abi.EXPORTED), declared ^ set(_abi.EXPORTED)
    lib = _abi.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.hsad_abi_version() == 1


def test_status_names_follow_errc():
    lib = _abi.lib()
    assert lib.hsad_status_name(13) == b"SingularAfterRidge"
    assert lib.hsad_status_name(16) == b"ConfigMismatch"
    assert lib.hsad_status_name(0) == b"Ok"
    assert lib.hsad_status_name(64) == b"CudaError"


def test_mirror_index_table():
    lib = _abi.lib()
    for (i, n), want in {(0, 5): 0, (4, 5): 4, (-1, 5): 1, (-2, 5): 2, (5, 5): 3, (6, 5): 2,
                         (9, 5): 1, (-7, 3): 1, (3, 1): 0}.items():
        assert lib.hsad_mirror_index(i, n) == want


def test_window_validation_messages(orc):
    lib = _abi.lib()
    for mode, a, b in ((0, 2, 0), (0, 1, 0), (1, 5, 5), (1, 5, 6), (1, 4, 9), (1, 0, 3)):
        w = _abi.Window(mode, a, a, b)
        st = lib.hsad_window_validate(C.byref(w))
        assert st == _abi.HSAD_E_INVALID_VALUE
        msg = lib.hsad_last_error_message().decode()
        with pytest.raises(orc.OracleError) as e:
            orc.port.window_validate(mode, a, b)
        assert msg == str(e.value)
    assert lib.hsad_window_validate(C.byref(_abi.Window(1, 0, 5, 13))) == 0


def test_daubechies_taps_equal_oracle(orc):
    lib = _abi.lib()
    for order in range(1, 11):
        low = (C.c_double * 20)(); high = (C.c_double * 20)(); n = C.c_int32()
        assert lib.hsad_daubechies_filters(order, low, high, C.byref(n)) == 0
        ol, oh = orc.port.daubechies(order)
        assert list(low[: n.value]) == list(ol) and list(high[: n.value]) == list(oh)
    assert lib.hsad_daubechies_filters(11, None, None, None) == _abi.HSAD_E_UNSUPPORTED_ORDER


def test_reduce_contract_errors_match_oracle(orc):
    """Argument errors are raised before any device work, like wavelet.cpp's probe."""
    import numpy as np
    lib = _abi.lib()
    cube = np.zeros((2, 2, 189))
    for order, target in ((0, 4), (11, 4), (2, 3), (2, 1), (2, 512), (10, 4)):
        st = lib.hsad_reduce(None, 8, 0, 0, 189, order, target, None, 8, None)
        with pytest.raises(orc.OracleError) as e:
            orc.port.reduce_cube(cube, order, target)
        assert st == e.value.code
        assert lib.hsad_last_error_message().decode() == str(e.value)


def test_strip_rows_and_quantum():
    lib = _abi.lib()
    req = (_abi.Request * 1)(_abi.Request(_abi.HSAD_DWRX, _abi.Window(1, 0, 5, 11), 1, 1e-6, 0.1,
                                          None, 8, None))
    r0 = C.c_int64(); n = C.c_int64()
    assert lib.hsad_strip_rows(100, 40, 60, req, 1, C.byref(r0), C.byref(n)) == 0
    assert (r0.value, n.value) == (35, 30)
    assert lib.hsad_strip_rows(100, 0, 10, req, 1, C.byref(r0), C.byref(n)) == 0
    assert (r0.value, n.value) == (0, 15)  # rows -5..-1 reflect onto 1..5
    q = lib.hsad_row_quantum(4096, 4096)
    assert q in (2, 4, 8, 16, 32, 64)


def test_decode_status():
    """Failure word: request position (bits 56..63), pixel (8..55), code (0..6) with
    the 0x80 "inverse overflowed" flag masked off."""
    lib = _abi.lib()
    e = _abi.PixelError()
    assert lib.hsad_decode_status((((7 * 100 + 3) << 8) | 13), 100, C.byref(e)) == 13
    assert (e.code, e.row, e.col) == (13, 7, 3)
    assert lib.hsad_decode_status((((7 * 100 + 3) << 8) | 13 | 0x80), 100, C.byref(e)) == 13
    assert (e.code, e.row, e.col) == (13, 7, 3)
    word = (5 << 56) | ((4095 * 4096 + 17) << 8) | 13
    assert lib.hsad_decode_status(word, 4096, C.byref(e)) == 13
    assert (e.code, e.row, e.col) == (13, 4095, 17)
    assert lib.hsad_decode_status(2**64 - 1, 100, C.byref(e)) == 0


def test_limits():
    lim = _abi.Limits()
    _abi.lib().hsad_get_limits(C.byref(lim))
    assert lim.max_detect_bands >= 4 and lim.max_window >= 21 and lim.max_reduce_bands >= 224


def test_pipeline_sharded_validates_on_host():
    lib = _abi.lib()
    req = (_abi.Request * 1)(_abi.Request(_abi.HSAD_LRX, _abi.Window(0, 5, 0, 0), 1, 1e-6, 0.1,
                                          None, 8, None))
    e = _abi.PixelError()
    assert lib.hsad_pipeline_sharded(None, 4, 4, 8, 2, 4, req, 1, 0, C.byref(e)) == _abi.HSAD_E_INVALID_VALUE
    assert lib.hsad_last_error_message() == b"InvalidValue: n_strips must be >= 1"


def test_fullband_gram_kernel_is_on_tcgen05():
    """SASS evidence: the full-band Gram kernel issues UTCIMMA (tcgen05.mma kind::i8) with
    TMEM loads, and no legacy mma.sync path stands in for it."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", "tc_gram_kernel", str(_abi.LIB_PATH)],
                          capture_output=True, text=True).stdout
    if "UTCIMMA" not in sass:  # older cuobjdump: no substring match for -fun
        sass = subprocess.run(["cuobjdump", "-sass", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "LDTM" in sass
