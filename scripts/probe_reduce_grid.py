"""Probe: K1 bandwidth when confined to n CTAs (1 CTA per SM): per-SM HBM pull rate."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows

cfg = CONFIGS["C5"]
rows = 1024
cube = generate_rows(rows, cfg["samples"], cfg["bands"], cfg["seed"], 0, rows, cfg["rate"], device="cuda")
out = torch.empty((rows, cfg["samples"], 4), dtype=torch.float64, device="cuda")
nbytes = cube.numel() * 4 + out.numel() * 8
for n in (8, 16, 24, 32, 48, 64, 96, 148):
    os.environ["HSAD_REDUCE_GRID"] = str(n)
    fn = lambda: hs._abi.lib().hsad_reduce(cube.data_ptr(), 4, rows, cfg["samples"], cfg["bands"], 2, 4, out.data_ptr(), 8, None)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(10): fn()
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"ctas {n:4d}  ms {ms:.3f}  GB/s {nbytes/ms/1e6:.0f}  per-SM GB/s {nbytes/ms/1e6/n:.1f}", flush=True)
