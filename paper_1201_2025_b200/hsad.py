"""Python mirror of the reference detector API over the B200 C-ABI.

Names, argument meaning and errors follow the reference's C++ API
(proj/core/include/hsad/{wavelet,detect}.hpp):

    daubechies_filters(order)                         wavelet.hpp:24
    reduce_cube(cube, filters|order, target_bands)    wavelet.hpp:55-56
    mirror_index(i, n)                                detect.hpp:68
    WindowConfig.single / .dual / validate / describe detect.hpp:20-33
    DetectOptions(ridge, dwest.eigen_fraction)        detect.hpp:35-45
    local_rx / dwrx / dwest / detect -> ScoreMap      detect.hpp:49-92

Cubes are CUDA tensors (torch is the device-memory plumbing) shaped
(lines, samples, bands), BIP, fp32 or fp64. Every call runs the sm_100a kernels
of libhsad_b200.so; a CPU tensor raises (no CPU fallback). Errors raise
HsadError carrying the reference's errc name and "at pixel (r, c)" suffix.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import _abi
from ._abi import HSAD_DWEST, HSAD_DWRX, HSAD_LRX, PixelError, Request, Window

ALGORITHMS = {"lrx": HSAD_LRX, "dwrx": HSAD_DWRX, "dwest": HSAD_DWEST}
ALGORITHM_NAMES = {v: k for k, v in ALGORITHMS.items()}


class HsadError(RuntimeError):
    """hsad::Error (error.hpp:36-45): what() = "<Name>: <message>"."""

    def __init__(self, code: int, message: str, row: int = -1, col: int = -1):
        super().__init__(message)
        self.code = code
        self.name = _abi.lib().hsad_status_name(code).decode()
        self.row, self.col = row, col


def _check(status: int, err: PixelError | None = None) -> None:
    if status != _abi.HSAD_OK:
        msg = _abi.lib().hsad_last_error_message().decode()
        row = err.row if err is not None else -1
        col = err.col if err is not None else -1
        raise HsadError(status, msg, row, col)


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA tensor: the hsad B200 path has no CPU fallback")
    if t.dtype not in (torch.float32, torch.float64):
        raise TypeError(f"{what} must be float32 or float64, got {t.dtype}")
    return t.contiguous()


# --------------------------------------------------------------------------- wavelet
@dataclass
class WaveletFilterPair:
    low: list
    high: list
    order: int

    def length(self) -> int:
        return len(self.low)


def daubechies_filters(order: int) -> WaveletFilterPair:
    low = (C.c_double * 32)(); high = (C.c_double * 32)(); n = C.c_int32(0)
    _check(_abi.lib().hsad_daubechies_filters(order, low, high, C.byref(n)))
    return WaveletFilterPair(list(low[: n.value]), list(high[: n.value]), order)


def reduce_cube(cube: torch.Tensor, filters: WaveletFilterPair | int = 2, target_bands: int = 4,
                workers: int = 1, out_dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """hsad::reduce_cube (wavelet.cpp:148-167) on the GPU. `workers` is accepted for
    signature parity; the GPU grid replaces the row threads."""
    order = filters.order if isinstance(filters, WaveletFilterPair) else int(filters)
    cube = _require_cuda(cube, "cube")
    lines, samples, bands = cube.shape
    out = torch.empty((lines, samples, max(target_bands, 0)), dtype=out_dtype, device=cube.device)
    _check(_abi.lib().hsad_reduce(cube.data_ptr(), cube.element_size(), lines, samples, bands,
                                  order, target_bands, out.data_ptr(), out.element_size(),
                                  _stream_ptr()))
    return out


# --------------------------------------------------------------------------- windows
@dataclass
class WindowConfig:
    mode: str = "single"  # "single" | "dual"
    single_size: int = 15
    inner_size: int = 5
    outer_size: int = 13

    @staticmethod
    def single(size: int) -> "WindowConfig":
        w = WindowConfig("single", single_size=size)
        w.validate()
        return w

    @staticmethod
    def dual(inner: int, outer: int) -> "WindowConfig":
        w = WindowConfig("dual", inner_size=inner, outer_size=outer)
        w.validate()
        return w

    def to_c(self) -> Window:
        return Window(_abi.WINDOW_SINGLE if self.mode == "single" else _abi.WINDOW_DUAL,
                      self.single_size, self.inner_size, self.outer_size)

    def validate(self) -> None:
        w = self.to_c()
        _check(_abi.lib().hsad_window_validate(C.byref(w)))

    def describe(self) -> str:
        return str(self.single_size) if self.mode == "single" else f"{self.inner_size}/{self.outer_size}"


def mirror_index(i: int, n: int) -> int:
    return _abi.lib().hsad_mirror_index(i, n)


@dataclass
class DwestConfig:
    eigen_fraction: float = 0.1


@dataclass
class DetectOptions:
    ridge: float = 1e-6
    dwest: DwestConfig = field(default_factory=DwestConfig)
    workers: int = 1
    guard: int = 1  # LRX guard box (extension; 1 = the reference)


@dataclass
class ScoreMap:
    lines: int = 0
    samples: int = 0
    scores: torch.Tensor | None = None  # (lines, samples) on the device
    algorithm: str = ""
    window: str = ""
    ridge: float = 0.0
    eigen_fraction: float = 0.0
    seconds: float = 0.0
    workers: int = 1
    eigcount: torch.Tensor | None = None  # DWEST extension, int8

    def at(self, row: int, col: int) -> float:
        return float(self.scores[row, col])


@dataclass
class DetectRequest:
    """One detector of a fused hsad_detect_multi call."""

    algorithm: str
    window: WindowConfig
    ridge: float = 1e-6
    eigen_fraction: float = 0.1
    guard: int = 1
    score_dtype: torch.dtype = torch.float64
    eigcount: bool = False


def _make_request(r: DetectRequest, scores: torch.Tensor, counts: torch.Tensor | None) -> Request:
    return Request(ALGORITHMS[r.algorithm], r.window.to_c(), r.guard, r.ridge, r.eigen_fraction,
                   scores.data_ptr(), scores.element_size(),
                   counts.data_ptr() if counts is not None else None)


def strip_rows(lines: int, row_begin: int, row_end: int, requests: Sequence[DetectRequest]):
    """Global rows [r0, r0 + n) that output rows [row_begin, row_end) read."""
    reqs = (Request * len(requests))(*[
        Request(ALGORITHMS[r.algorithm], r.window.to_c(), r.guard, r.ridge, r.eigen_fraction,
                None, 8, None) for r in requests])
    r0 = C.c_int64(0); n = C.c_int64(0)
    _check(_abi.lib().hsad_strip_rows(lines, row_begin, row_end, reqs, len(requests),
                                      C.byref(r0), C.byref(n)))
    return r0.value, n.value


def row_quantum(lines: int, samples: int) -> int:
    return int(_abi.lib().hsad_row_quantum(lines, samples))


def detect_multi(cube: torch.Tensor, requests: Sequence[DetectRequest], *, lines: int | None = None,
                 buf_row0: int = 0, row_begin: int | None = None, row_end: int | None = None,
                 status: torch.Tensor | None = None, outputs=None):
    """Fused hsad_detect_multi: all requests share one pass of window statistics.

    `cube` holds global rows [buf_row0, buf_row0 + cube.shape[0]) of an image with
    `lines` rows (default: the cube is the whole image). Returns a list of
    (scores, eigcount-or-None) tensors covering rows [row_begin, row_end). With a
    device `status` tensor (uint64 view, 1 element, initialised to all ones) the
    call is asynchronous and per-pixel failures are recorded there.
    """
    cube = _require_cuda(cube, "cube")
    buf_rows, samples, bands = cube.shape
    lines = buf_rows if lines is None else lines
    rb = 0 if row_begin is None else row_begin
    re = lines if row_end is None else row_end
    if outputs is None:
        outputs = []
        for r in requests:
            sc = torch.empty((re - rb, samples), dtype=r.score_dtype, device=cube.device)
            cnt = (torch.empty((re - rb, samples), dtype=torch.int8, device=cube.device)
                   if (r.eigcount and r.algorithm == "dwest") else None)
            outputs.append((sc, cnt))
    reqs = (Request * len(requests))(*[
        _make_request(r, sc, cnt) for r, (sc, cnt) in zip(requests, outputs)])
    err = PixelError()
    st = _abi.lib().hsad_detect_multi(cube.data_ptr(), cube.element_size(), lines, samples, bands,
                                      buf_row0, buf_rows, rb, re, reqs, len(requests),
                                      status.data_ptr() if status is not None else None,
                                      C.byref(err), _stream_ptr())
    _check(st, err)
    return outputs


def reduce_detect(cube: torch.Tensor, requests: Sequence[DetectRequest],
                  filters: WaveletFilterPair | int = 2, target_bands: int = 4, *,
                  lines: int | None = None, buf_row0: int = 0, row_begin: int | None = None,
                  row_end: int | None = None, status: torch.Tensor | None = None,
                  reduced: torch.Tensor | None = None, outputs=None):
    """hsad_reduce_detect: reduce_cube followed by detect_multi in one launch.

    `cube` is the fp32 full-band cube (rows [buf_row0, buf_row0 + cube.shape[0]) of an
    image with `lines` rows). Returns (reduced, outputs): the fp64 reduced cube of the
    same rows and the per-request (scores, eigcount-or-None) list of detect_multi.
    """
    cube = _require_cuda(cube, "cube")
    if cube.dtype != torch.float32:
        raise HsadError(_abi.HSAD_E_INVALID_VALUE, "InvalidValue: reduce_detect takes an fp32 cube")
    cube = cube.contiguous()
    order = filters.order if isinstance(filters, WaveletFilterPair) else int(filters)
    buf_rows, samples, bands = cube.shape
    lines = buf_rows if lines is None else lines
    rb = 0 if row_begin is None else row_begin
    re = lines if row_end is None else row_end
    if reduced is None:
        reduced = torch.empty((buf_rows, samples, max(target_bands, 0)), dtype=torch.float64,
                              device=cube.device)
    if outputs is None:
        outputs = []
        for r in requests:
            sc = torch.empty((max(re - rb, 0), samples), dtype=r.score_dtype, device=cube.device)
            cnt = (torch.empty((max(re - rb, 0), samples), dtype=torch.int8, device=cube.device)
                   if (r.eigcount and r.algorithm == "dwest") else None)
            outputs.append((sc, cnt))
    reqs = (Request * len(requests))(*[
        _make_request(r, sc, cnt) for r, (sc, cnt) in zip(requests, outputs)])
    err = PixelError()
    st = _abi.lib().hsad_reduce_detect(cube.data_ptr(), lines, samples, bands, order, target_bands,
                                       buf_row0, buf_rows, rb, re, reduced.data_ptr(), reqs,
                                       len(requests),
                                       status.data_ptr() if status is not None else None,
                                       C.byref(err), _stream_ptr())
    _check(st, err)
    return reduced, outputs


def _single(cube: torch.Tensor, algorithm: str, window: WindowConfig, ridge: float,
            eigen_fraction: float, guard: int = 1, score_dtype=torch.float64) -> ScoreMap:
    cube = _require_cuda(cube, "cube")
    lines, samples, _ = cube.shape
    t0 = time.perf_counter()
    req = DetectRequest(algorithm, window, ridge=ridge, eigen_fraction=eigen_fraction, guard=guard,
                        score_dtype=score_dtype, eigcount=algorithm == "dwest")
    # hsad_detect is synchronous (detect.hpp:91-92 semantics)
    scores, counts = detect_multi(cube, [req])[0]
    torch.cuda.current_stream().synchronize()
    m = ScoreMap(lines, samples, scores, algorithm, window.describe(), seconds=0.0)
    if algorithm in ("lrx", "dwrx"):
        m.ridge = ridge
    else:
        m.eigen_fraction = eigen_fraction
    m.eigcount = counts
    m.seconds = time.perf_counter() - t0
    return m


def _require_mode(window: WindowConfig, mode: str, algo: str) -> None:
    window.validate()
    if window.mode != mode:
        raise HsadError(_abi.HSAD_E_CONFIG_MISMATCH,
                        f"ConfigMismatch: {algo} requires a {mode} window")


def local_rx(cube: torch.Tensor, config: WindowConfig, ridge: float = 1e-6, workers: int = 1,
             guard: int = 1) -> ScoreMap:
    _require_mode(config, "single", "local_rx")
    m = _single(cube, "lrx", config, ridge, 0.0, guard)
    m.workers = workers
    return m


def dwrx(cube: torch.Tensor, config: WindowConfig, ridge: float = 1e-6, workers: int = 1) -> ScoreMap:
    _require_mode(config, "dual", "dwrx")
    m = _single(cube, "dwrx", config, ridge, 0.0)
    m.workers = workers
    return m


def dwest(cube: torch.Tensor, config: WindowConfig, dcfg: DwestConfig | float = DwestConfig(),
          workers: int = 1) -> ScoreMap:
    _require_mode(config, "dual", "dwest")
    frac = dcfg.eigen_fraction if isinstance(dcfg, DwestConfig) else float(dcfg)
    if not (0.0 < frac <= 1.0):
        raise HsadError(_abi.HSAD_E_INVALID_VALUE, "InvalidValue: eigen fraction must be in (0, 1]")
    m = _single(cube, "dwest", config, 0.0, frac)
    m.workers = workers
    return m


def dwest_pairs(cdiff: torch.Tensor, mdiff: torch.Tensor, eigen_fraction: float = 0.1):
    """symmetric_eigen + the DWEST selection (stats.cpp:64-89, detect.cpp:252-263) on a batch
    of 4 x 4 matrices: cdiff (n, 4, 4) fp64 symmetric, mdiff (n, 4) fp64, CUDA tensors.
    Returns (scores fp64 (n,), counts int8 (n,), route int8 (n,): 0 = two-pair route,
    1 = general Jacobi route). The device code is the fused detectors'."""
    cdiff = _require_cuda(cdiff, "cdiff")
    mdiff = _require_cuda(mdiff, "mdiff")
    if cdiff.dtype != torch.float64 or mdiff.dtype != torch.float64:
        raise TypeError("dwest_pairs takes float64 tensors")
    n = cdiff.shape[0]
    if tuple(cdiff.shape[1:]) != (4, 4) or tuple(mdiff.shape) != (n, 4):
        raise ValueError("cdiff must be (n, 4, 4) and mdiff (n, 4)")
    scores = torch.empty(n, dtype=torch.float64, device=cdiff.device)
    counts = torch.empty(n, dtype=torch.int8, device=cdiff.device)
    route = torch.empty(n, dtype=torch.int8, device=cdiff.device)
    _check(_abi.lib().hsad_dwest_pairs(cdiff.data_ptr(), mdiff.data_ptr(), n, float(eigen_fraction),
                                       scores.data_ptr(), counts.data_ptr(), route.data_ptr(),
                                       _stream_ptr()))
    return scores, counts, route


def dual_window_samples(cube: torch.Tensor, row: int, col: int, config: WindowConfig):
    """hsad::dual_window_samples (detect.cpp:150-157): (inner, outer) sample sets of one pixel as
    (count, bands) fp64 tensors in the reference's scan order (= SampleSet::vectors transposed)."""
    cube = _require_cuda(cube, "cube")
    lines, samples, bands = cube.shape
    win = config.to_c()
    n_in = max(config.inner_size, 0) ** 2
    n_out = max(max(config.outer_size, 0) ** 2 - n_in, 0)
    inner = torch.empty((n_in, bands), dtype=torch.float64, device=cube.device)
    outer = torch.empty((n_out, bands), dtype=torch.float64, device=cube.device)
    _check(_abi.lib().hsad_dual_window_samples(cube.data_ptr(), cube.element_size(), lines, samples, bands,
                                               int(row), int(col), C.byref(win), inner.data_ptr(),
                                               outer.data_ptr(), _stream_ptr()))
    return inner, outer


def encode_score_map(scores: torch.Tensor) -> torch.Tensor:
    """The .raw payload of save_score_map (detect.cpp:291-318): little-endian fp32, as uint8."""
    scores = _require_cuda(scores, "scores")
    raw = torch.empty(scores.numel() * 4, dtype=torch.uint8, device=scores.device)
    _check(_abi.lib().hsad_encode_score_map(scores.data_ptr(), scores.element_size(), scores.numel(),
                                            raw.data_ptr(), _stream_ptr()))
    return raw


def save_score_map(score_map: "ScoreMap", prefix) -> None:
    """hsad::save_score_map (detect.cpp:291-318): <prefix>.hdr (ENVI text, cube.cpp:184-196) and
    <prefix>.raw (1 band, BSQ, data type 4, little-endian), the payload encoded on the device."""
    from pathlib import Path
    prefix = Path(prefix)
    hdr = ("ENVI\n" f"samples = {score_map.samples}\n" f"lines = {score_map.lines}\n" "bands = 1\n"
           "header offset = 0\n" "file type = ENVI Standard\n" "data type = 4\n"
           "interleave = bsq\n" "byte order = 0\n")
    try:
        prefix.with_suffix(".hdr").write_text(hdr)
        prefix.with_suffix(".raw").write_bytes(encode_score_map(score_map.scores).cpu().numpy().tobytes())
    except OSError as e:
        raise HsadError(_abi.HSAD_E_IO_FAILURE, f"IoFailure: cannot open {e.filename} for writing") from e


def detect(cube: torch.Tensor, algorithm: str, config: WindowConfig,
           options: DetectOptions = DetectOptions()) -> ScoreMap:
    """hsad::detect dispatch (detect.cpp:278-289)."""
    if algorithm == "lrx":
        return local_rx(cube, config, options.ridge, options.workers, options.guard)
    if algorithm == "dwrx":
        return dwrx(cube, config, options.ridge, options.workers)
    if algorithm == "dwest":
        return dwest(cube, config, options.dwest, options.workers)
    raise HsadError(_abi.HSAD_E_INVALID_VALUE, f"InvalidValue: unknown algorithm '{algorithm}'")


def pipeline_host(h_cube, order: int, target_bands: int, requests: Sequence[DetectRequest],
                  outputs):
    """hsad_pipeline_host: host fp32 cube -> H2D -> reduce -> fused detectors -> D2H.

    `h_cube` is a CPU float32 tensor (pinned recommended); `outputs` a list of
    (scores, eigcount-or-None) CPU tensors sized (lines, samples)."""
    lines, samples, bands = h_cube.shape
    reqs = (Request * len(requests))(*[
        _make_request(r, sc, cnt) for r, (sc, cnt) in zip(requests, outputs)])
    err = PixelError()
    st = _abi.lib().hsad_pipeline_host(h_cube.data_ptr(), lines, samples, bands, order,
                                       target_bands, reqs, len(requests), C.byref(err),
                                       _stream_ptr())
    _check(st, err)
    return outputs
