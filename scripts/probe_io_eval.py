"""Probe: C5-scale throughput of the ingest / evaluation kernels (csrc/ingest.cu, csrc/eval.cu).

BSQ / BIL fp32 raw cube (4096 x 4096 x 224, 15 GB) -> BIP fp32 and fp64; exact ROC
(AUC only and with all points), top-k, adaptive threshold, PGM stretch on a 4096^2
fp64 score map with a 0.1% truth mask. CUDA events, median of 5 after warm-up.
"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1201_2025_b200 import evalio


def timeit(fn, n=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(n):
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


L, S, B = 4096, 4096, 224
out = {}
raw = torch.empty(L * S * B * 4, dtype=torch.uint8, device="cuda")
raw.view(torch.float32).normal_()
for il in ("bsq", "bil"):
    hdr = evalio.CubeHeader(S, L, B, il, 4, 0)
    for dt, eb in ((torch.float32, 4), (torch.float64, 8)):
        cube = torch.empty((L, S, B), dtype=dt, device="cuda")
        from paper_1201_2025_b200 import _abi
        import ctypes as C
        h = hdr.to_c()
        fn = lambda: _abi.lib().hsad_read_cube(raw.data_ptr(), raw.numel(), C.byref(h), cube.data_ptr(), eb,
                                              torch.cuda.current_stream().cuda_stream)
        ms = timeit(fn)
        gb = (raw.numel() + cube.numel() * eb) / 1e9
        out[f"read_cube {il} f32->{'f32' if eb == 4 else 'f64'}"] = {"ms": ms, "GB": gb, "GB/s": gb / ms * 1e3}
        del cube
# fused decode + DWT from the raw BSQ / BIL bytes vs read_cube then reduce_cube
import ctypes as C
from paper_1201_2025_b200 import _abi
red = torch.empty((L, S, 4), dtype=torch.float64, device="cuda")
for il in ("bsq", "bil"):
    h = evalio.CubeHeader(S, L, B, il, 4, 0).to_c()
    fn = lambda: _abi.lib().hsad_reduce_raw(raw.data_ptr(), raw.numel(), C.byref(h), 2, 4, red.data_ptr(), 8,
                                            torch.cuda.current_stream().cuda_stream)
    ms = timeit(fn)
    gb = (raw.numel() + red.numel() * 8) / 1e9
    out[f"reduce_raw {il} f32 -> 4 bands f64"] = {"ms": ms, "GB": gb, "GB/s": gb / ms * 1e3}
del raw, red
torch.cuda.empty_cache()
g = torch.Generator(device="cuda").manual_seed(7)
scores = torch.empty((L, S), dtype=torch.float64, device="cuda").exponential_(generator=g)
truth = (torch.rand((L, S), device="cuda", generator=g) < 0.001).to(torch.uint8)
n = L * S
k = int(truth.sum())
out["roc auc-only"] = {"ms": timeit(lambda: evalio.roc_curve(scores, truth, points=False))}
out["roc with points"] = {"ms": timeit(lambda: evalio.roc_curve(scores, truth))}
out["top_k"] = {"ms": timeit(lambda: evalio.top_k(scores, k)), "k": k}
out["adaptive_threshold"] = {"ms": timeit(lambda: evalio.adaptive_threshold(scores, 3.0))}
px = torch.empty(n, dtype=torch.uint8, device="cuda")
out["render_pgm (device pixels)"] = {"ms": timeit(lambda: _abi.lib().hsad_render_pgm(
    scores.data_ptr(), 8, n, px.data_ptr(), torch.cuda.current_stream().cuda_stream))}
out["_note"] = "4096x4096 maps, truth 0.1%; each call synchronous (includes its small D2H reads)"
print(json.dumps(out, indent=1))
