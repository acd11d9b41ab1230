"""Probe: hsad_reduce_raw on a C5-sized raw fp32 BSQ / BIL cube (HSAD_B200_LIB selects the build)."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1201_2025_b200 import _abi, evalio
L, S, B = 4096, 4096, 224
raw = torch.empty(L * S * B * 4, dtype=torch.uint8, device="cuda")
raw.view(torch.float32).normal_()
red = torch.empty((L, S, 4), dtype=torch.float64, device="cuda")
for il in ("bsq", "bil"):
    h = evalio.CubeHeader(S, L, B, il, 4, 0).to_c()
    fn = lambda: _abi.lib().hsad_reduce_raw(raw.data_ptr(), raw.numel(), C.byref(h), 2, 4, red.data_ptr(), 8,
                                            torch.cuda.current_stream().cuda_stream)
    for _ in range(2): assert fn() == 0
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ms = sorted(ts)[2]
    print(f"{Path(os.environ.get('HSAD_B200_LIB', 'default')).name} {il}: {ms:.3f} ms  {(raw.numel() + red.numel() * 8) / ms / 1e6:.0f} GB/s", flush=True)
