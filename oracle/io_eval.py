"""TEST INFRASTRUCTURE ONLY — CPU oracle for the ingest / evaluation rows.

* ``read_cube`` / ``roc_curve`` / ``adaptive_threshold`` / ``render_pgm``: numpy
  restatements of proj/core/src/cube.cpp:198-253 and proj/core/src/eval.cpp:10-109
  (same operation order where it decides the result: sequential sums for the
  threshold, exact integer AUC, round-half-away-from-zero for the PGM stretch);
* ``RefIO``: the reference's own cube.cpp / eval.cpp / pgm.cpp compiled in place
  (oracle/_ref/libhsad_ref_io.so, see oracle/Makefile) — the pin for the above.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import ERRC_NAMES, OracleError

HERE = Path(__file__).resolve().parent
REF_IO_SO = HERE / "_ref" / "libhsad_ref_io.so"

_DT = {1: np.uint8, 2: np.int16, 4: np.float32, 5: np.float64, 12: np.uint16}
_IL = {"bsq": 0, "bil": 1, "bip": 2}


def element_size(code: int) -> int:  # cube.cpp:22-33
    if code not in _DT:
        raise OracleError(2, f"InvalidValue: unsupported data type code {code}")
    return np.dtype(_DT[code]).itemsize


def read_cube(raw: bytes | np.ndarray, samples: int, lines: int, bands: int, interleave: str,
              data_type_code: int, byte_order: int) -> np.ndarray:
    """cube.cpp:198-253 -> (lines, samples, bands) fp64 BIP."""
    if samples < 1 or lines < 1 or bands < 1:  # cube.cpp:39-45
        raise OracleError(2, "InvalidValue: samples, lines and bands must all be >= 1")
    es = element_size(data_type_code)
    if byte_order not in (0, 1):
        raise OracleError(2, "InvalidValue: byte order must be 0 or 1")
    raw = np.frombuffer(bytes(raw) if not isinstance(raw, np.ndarray) else raw.tobytes(), np.uint8)
    expected = samples * lines * bands * es
    if raw.size != expected:
        raise OracleError(3, f"SizeMismatch: raw data is {raw.size} bytes, header expects {expected}")
    dt = np.dtype(_DT[data_type_code]).newbyteorder(">" if byte_order == 1 else "<")
    v = np.frombuffer(raw.tobytes(), dt).astype(np.float64)
    if interleave == "bsq":
        cube = v.reshape(bands, lines, samples).transpose(1, 2, 0)
    elif interleave == "bil":
        cube = v.reshape(lines, bands, samples).transpose(0, 2, 1)
    else:
        cube = v.reshape(lines, samples, bands)
    cube = np.ascontiguousarray(cube)
    bad = ~np.isfinite(cube)
    if bad.any():  # first in (row, col, band) order, cube.cpp:244-247
        r, c, b = np.unravel_index(int(np.flatnonzero(bad.ravel())[0]), cube.shape)
        raise OracleError(4, f"NonFiniteValue: at (row={r}, col={c}, band={b})")
    return cube


def roc_curve(scores: np.ndarray, truth: np.ndarray):
    """eval.cpp:10-57 -> (far, td, auc, auc_twice_num)."""
    s = np.asarray(scores, np.float64).ravel()
    t = np.asarray(truth).ravel() != 0
    pos = int(t.sum())
    neg = s.size - pos
    if pos == 0 or neg == 0:
        raise OracleError(20, "DegenerateTruth: truth mask must contain both classes")
    s = np.where(s == 0.0, 0.0, s)  # -0.0 == 0.0 in the reference's == grouping
    order = np.argsort(-s, kind="stable")
    ss, tt = s[order], t[order]
    heads = np.flatnonzero(np.r_[True, ss[1:] != ss[:-1]])
    tp_step = np.add.reduceat(tt.astype(np.uint64), heads)
    cnt = np.diff(np.r_[heads, ss.size]).astype(np.uint64)
    fp_step = cnt - tp_step
    tp_before = np.r_[np.uint64(0), np.cumsum(tp_step)[:-1]].astype(np.uint64)
    num = int(np.sum(fp_step * (np.uint64(2) * tp_before + tp_step), dtype=np.uint64))
    tp, fp = np.cumsum(tp_step), np.cumsum(fp_step)
    far = np.r_[0.0, fp.astype(np.float64) / float(neg)]
    td = np.r_[0.0, tp.astype(np.float64) / float(pos)]
    return far, td, num / (2.0 * float(pos) * float(neg)), num


def adaptive_threshold(scores: np.ndarray, z_alpha: float):
    """eval.cpp:69-90 with the reference's sequential sums (np.add.accumulate is
    a left-to-right loop, unlike np.sum's pairwise summation)."""
    s = np.asarray(scores, np.float64).ravel()
    if s.size == 0:
        raise OracleError(2, "InvalidValue: cannot threshold an empty score map")
    n = float(s.size)
    mean = np.add.accumulate(s)[-1] / n
    d = s - mean
    var = np.add.accumulate(d * d)[-1] / n
    tau = mean + z_alpha * np.sqrt(var)
    return tau, (s > tau).astype(np.uint8)


def render_pgm(scores: np.ndarray) -> bytes:
    """eval.cpp:92-109 + pgm.cpp encode: min-max stretch, lround (half away from zero)."""
    s = np.asarray(scores, np.float64)
    lines, samples = s.shape
    flat = s.ravel()
    px = np.zeros(flat.size, np.uint8)
    lo, hi = (flat.min(), flat.max()) if flat.size else (0.0, 0.0)
    if hi > lo:
        x = (flat - lo) * (255.0 / (hi - lo))
        fl = np.floor(x)
        px = np.where(x - fl >= 0.5, fl + 1.0, fl).astype(np.uint8)
    return f"P5\n{samples} {lines}\n255\n".encode() + px.tobytes()


class RefIO:
    """ctypes over oracle/_ref/libhsad_ref_io.so (the reference's own code)."""

    def __init__(self, path: Path = REF_IO_SO):
        lib = C.CDLL(str(path))
        P, U8, D, L, I = C.POINTER, C.c_void_p, C.c_void_p, C.c_long, C.c_int
        lib.refio_last_error.restype = C.c_char_p
        lib.refio_read_cube.argtypes = [U8, L, I, I, I, I, I, I, D]
        lib.refio_roc.argtypes = [D, U8, I, I, D, D, L, P(L), P(C.c_double)]
        lib.refio_threshold.argtypes = [D, I, I, C.c_double, P(C.c_double), U8]
        lib.refio_render_pgm.argtypes = [D, I, I, U8, L, P(L)]
        self.lib = lib

    def _err(self, st):
        if st:
            raise OracleError(st, self.lib.refio_last_error().decode())

    def read_cube(self, raw, samples, lines, bands, interleave, code, byte_order):
        raw = np.frombuffer(bytes(raw), np.uint8).copy()
        out = np.empty((max(lines, 1), max(samples, 1), max(bands, 1)), np.float64)
        il = _IL[interleave] if isinstance(interleave, str) else interleave
        self._err(self.lib.refio_read_cube(raw.ctypes.data, raw.size, samples, lines, bands, il, code,
                                           byte_order, out.ctypes.data))
        return out

    def roc_curve(self, scores, truth):
        s = np.ascontiguousarray(scores, np.float64)
        t = np.ascontiguousarray(truth, np.uint8)
        cap = s.size + 1
        far, td = np.empty(cap), np.empty(cap)
        n, a = C.c_long(0), C.c_double(0.0)
        self._err(self.lib.refio_roc(s.ctypes.data, t.ctypes.data, s.shape[0], s.shape[1],
                                     far.ctypes.data, td.ctypes.data, cap, C.byref(n), C.byref(a)))
        return far[: n.value], td[: n.value], a.value

    def adaptive_threshold(self, scores, z):
        s = np.ascontiguousarray(scores, np.float64)
        mask = np.empty(s.size, np.uint8)
        tau = C.c_double(0.0)
        self._err(self.lib.refio_threshold(s.ctypes.data, s.shape[0], s.shape[1], z, C.byref(tau),
                                           mask.ctypes.data))
        return tau.value, mask

    def render_pgm(self, scores):
        s = np.ascontiguousarray(scores, np.float64)
        out = np.empty(s.size + 64, np.uint8)
        n = C.c_long(0)
        self._err(self.lib.refio_render_pgm(s.ctypes.data, s.shape[0], s.shape[1], out.ctypes.data,
                                            out.size, C.byref(n)))
        return out[: n.value].tobytes()


def ref_io() -> RefIO | None:
    return RefIO() if REF_IO_SO.exists() else None


__all__ = ["read_cube", "roc_curve", "adaptive_threshold", "render_pgm", "RefIO", "ref_io", "ERRC_NAMES"]
