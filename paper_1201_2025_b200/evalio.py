"""Python mirror of the reference's cube ingest and evaluation API over the C-ABI.

    read_cube(raw, header)            hsad::read_cube          cube.hpp:70-72, cube.cpp:198-253
    reduce_raw(raw, header, order, t) read_cube + reduce_cube  (wavelet.cpp:148-167), one pass
    pipeline_raw(host_raw, header, ...) read + reduce + detect from HOST raw bytes (streamed)
    roc_curve(scores, truth)          hsad::roc_curve          eval.hpp:23, eval.cpp:10-57
    auc(curve)                        hsad::auc                eval.hpp:26, eval.cpp:59-67
    adaptive_threshold(scores, z)     hsad::adaptive_threshold eval.hpp:37, eval.cpp:69-90
    render_pgm(scores)                hsad::render_pgm         eval.hpp:41, eval.cpp:92-110
    top_k(scores, k)                  the parity gate's top-k anomaly set

Inputs and outputs are CUDA tensors (score maps (lines, samples) fp64 or fp32,
truth masks uint8); the work runs in libhsad_b200.so (csrc/ingest.cu,
csrc/eval.cu). Errors raise HsadError with the reference's errc names.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _abi
from ._abi import CubeHeader as _CHeader, RocSummary
from .hsad import HsadError, ScoreMap, _check, _stream_ptr

INTERLEAVE = {"bsq": _abi.HSAD_BSQ, "bil": _abi.HSAD_BIL, "bip": _abi.HSAD_BIP}


@dataclass
class CubeHeader:
    """hsad::CubeHeader (cube.hpp:26-37)."""
    samples: int = 0
    lines: int = 0
    bands: int = 0
    interleave: str = "bsq"
    data_type_code: int = 5
    byte_order: int = 0

    def to_c(self) -> _CHeader:
        il = INTERLEAVE.get(self.interleave, -1) if isinstance(self.interleave, str) else int(self.interleave)
        return _CHeader(self.samples, self.lines, self.bands, il, self.data_type_code, self.byte_order)


def _u8(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA tensor: the hsad B200 path has no CPU fallback")
    return t.contiguous()


def read_cube(raw: torch.Tensor, header: CubeHeader, out_dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """Decode raw ENVI bytes (a CUDA uint8 tensor) into a (lines, samples, bands) BIP cube."""
    raw = _u8(raw, "raw")
    h = header.to_c()
    shape = (max(header.lines, 0), max(header.samples, 0), max(header.bands, 0))
    out = torch.empty(shape, dtype=out_dtype, device=raw.device)
    _check(_abi.lib().hsad_read_cube(raw.data_ptr(), raw.numel() * raw.element_size(), C.byref(h),
                                     out.data_ptr(), out.element_size(), _stream_ptr()))
    return out


def reduce_raw(raw: torch.Tensor, header: CubeHeader, order: int = 2, target_bands: int = 4,
               out_dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """read_cube + reduce_cube in one pass over a raw BSQ / BIL cube (no BIP intermediate)."""
    raw = _u8(raw, "raw")
    h = header.to_c()
    out = torch.empty((max(header.lines, 0), max(header.samples, 0), max(target_bands, 0)),
                      dtype=out_dtype, device=raw.device)
    _check(_abi.lib().hsad_reduce_raw(raw.data_ptr(), raw.numel() * raw.element_size(), C.byref(h),
                                      order, target_bands, out.data_ptr(), out.element_size(),
                                      _stream_ptr()))
    return out


def pipeline_raw(h_raw, header: CubeHeader, order: int, target_bands: int, requests, outputs):
    """hsad_pipeline_raw: raw ENVI bytes on the HOST (numpy array / CPU uint8 tensor, pinned
    recommended) -> streamed decode + DWT + detectors -> host maps. `outputs` is a list of
    (scores, eigcount-or-None) CPU tensors sized (lines, samples)."""
    from ._abi import PixelError, Request
    from .hsad import _make_request
    buf = h_raw if isinstance(h_raw, torch.Tensor) else torch.from_numpy(h_raw)
    if buf.is_cuda:
        raise TypeError("h_raw must be host memory (use reduce_raw for device buffers)")
    buf = buf.contiguous()
    h = header.to_c()
    reqs = (Request * len(requests))(*[_make_request(r, sc, cnt) for r, (sc, cnt) in zip(requests, outputs)])
    err = PixelError()
    _check(_abi.lib().hsad_pipeline_raw(buf.data_ptr(), buf.numel() * buf.element_size(), C.byref(h), order,
                                        target_bands, reqs, len(requests), C.byref(err), _stream_ptr()), err)
    return outputs


def _scores(s) -> torch.Tensor:
    t = s.scores if isinstance(s, ScoreMap) else s
    t = _u8(t, "scores")
    if t.dtype not in (torch.float64, torch.float32):
        raise TypeError("scores must be float64 or float32")
    return t


@dataclass
class RocCurve:
    """hsad::RocCurve (eval.hpp:17-20): far/td points on the device, exact auc."""
    far: torch.Tensor | None = None
    td: torch.Tensor | None = None
    auc: float = 0.0
    positives: int = 0
    negatives: int = 0
    auc_twice_num: int = 0

    @property
    def points(self):
        return list(zip(self.far.tolist(), self.td.tolist()))


def roc_curve(scores, truth: torch.Tensor, points: bool = True) -> RocCurve:
    s = _scores(scores)
    t = _u8(truth, "truth")
    if tuple(s.shape) != tuple(t.shape):  # eval.cpp:11-15
        raise HsadError(_abi.HSAD_E_DIMENSION_MISMATCH,
                        f"DimensionMismatch: score map is {s.shape[0]}x{s.shape[1]}, truth is "
                        f"{t.shape[0]}x{t.shape[1]}")
    if t.dtype != torch.uint8:
        t = (t != 0).to(torch.uint8)
    n = s.numel()
    summ = RocSummary()
    if not points:
        _check(_abi.lib().hsad_roc(s.data_ptr(), s.element_size(), t.data_ptr(), n, C.byref(summ),
                                   None, None, 0, _stream_ptr()))
        return RocCurve(None, None, summ.auc, summ.positives, summ.negatives, summ.auc_twice_num)
    far = torch.empty(n + 1, dtype=torch.float64, device=s.device)
    td = torch.empty(n + 1, dtype=torch.float64, device=s.device)
    _check(_abi.lib().hsad_roc(s.data_ptr(), s.element_size(), t.data_ptr(), n, C.byref(summ),
                               far.data_ptr(), td.data_ptr(), n + 1, _stream_ptr()))
    k = int(summ.distinct) + 1
    return RocCurve(far[:k], td[:k], summ.auc, summ.positives, summ.negatives, summ.auc_twice_num)


def auc(curve: RocCurve) -> float:
    """Trapezoidal area under the curve's points (eval.cpp:59-67), on the host."""
    far, td = curve.far.cpu().tolist(), curve.td.cpu().tolist()
    area = 0.0
    for i in range(1, len(far)):
        area += (far[i] - far[i - 1]) * (td[i - 1] + td[i]) / 2.0
    return area


@dataclass
class ThresholdResult:
    tau: float = 0.0
    mask: torch.Tensor | None = None
    z_alpha: float = 0.0


def adaptive_threshold(scores, z_alpha: float) -> ThresholdResult:
    s = _scores(scores)
    mask = torch.empty(s.shape, dtype=torch.uint8, device=s.device)
    tau = C.c_double(0.0)
    _check(_abi.lib().hsad_adaptive_threshold(s.data_ptr(), s.element_size(), s.numel(), z_alpha,
                                              C.byref(tau), mask.data_ptr(), _stream_ptr()))
    return ThresholdResult(tau.value, mask, z_alpha)


def render_pgm(scores) -> bytes:
    """Complete PGM bytes: "P5\\n<w> <h>\\n255\\n" + the device-stretched pixels (pgm.cpp)."""
    s = _scores(scores)
    lines, samples = (s.shape[0], s.shape[1]) if s.dim() == 2 else (1, s.numel())
    px = torch.empty(s.numel(), dtype=torch.uint8, device=s.device)
    _check(_abi.lib().hsad_render_pgm(s.data_ptr(), s.element_size(), s.numel(), px.data_ptr(),
                                      _stream_ptr()))
    return f"P5\n{samples} {lines}\n255\n".encode() + px.cpu().numpy().tobytes()


def top_k(scores, k: int):
    """(ascending pixel indices of the k largest scores, k-th score); ties -> lower index."""
    s = _scores(scores)
    idx = torch.empty(k, dtype=torch.int64, device=s.device)
    kth = C.c_double(0.0)
    _check(_abi.lib().hsad_top_k(s.data_ptr(), s.element_size(), s.numel(), k, idx.data_ptr(),
                                 C.byref(kth), _stream_ptr()))
    return idx, kth.value
