"""B200-native (sm_100a) hsad hot path: db-N spectral DWT + LRX / DWRX / DWEST.

The product is libhsad_b200.so (C-ABI: include/hsad_gpu.h, kernels in csrc/).
This package holds its Python binding (`_abi`), the Python mirror of the
reference's detector API (`hsad`) and the row-strip multi-GPU driver
(`sharded`). Import fails loudly if the CUDA library has not been built.
"""
from . import _abi
from .hsad import (DetectOptions, DetectRequest, DwestConfig, HsadError, ScoreMap,
                   WaveletFilterPair, WindowConfig, daubechies_filters, detect, detect_multi, reduce_detect,
                   dual_window_samples, dwest, dwest_pairs, dwrx, encode_score_map, local_rx, mirror_index, pipeline_host, reduce_cube, row_quantum,
                   save_score_map, strip_rows)

_abi.lib()  # no CPU fallback: fail at import when libhsad_b200.so is missing

__all__ = [
    "DetectOptions", "DetectRequest", "DwestConfig", "HsadError", "ScoreMap", "WaveletFilterPair",
    "WindowConfig", "daubechies_filters", "detect", "detect_multi", "reduce_detect", "dual_window_samples", "dwest", "dwest_pairs", "dwrx", "encode_score_map", "local_rx",
    "mirror_index", "pipeline_host", "reduce_cube", "row_quantum", "save_score_map", "strip_rows",
]
