"""Probe: one C5 detector launch (LRX + DWRX + DWEST at one window pair) for ncu captures.

    python scripts/probe_one.py [inner outer] [reps]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows

inner = int(sys.argv[1]) if len(sys.argv) > 2 else 5
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 11
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"],
                     cfg["rate"], device="cuda")
red = hs.reduce_cube(cube, 2, 4)
del cube
torch.cuda.empty_cache()
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
reqs = [hs.DetectRequest("lrx", W1(outer)), hs.DetectRequest("dwrx", W2(inner, outer)),
        hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)]
st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
outs = hs.detect_multi(red, reqs, status=st)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
for _ in range(reps):
    s.record()
    hs.detect_multi(red, reqs, status=st, outputs=outs)
    e.record()
    e.synchronize()
    print(f"{inner}/{outer} detect ms {s.elapsed_time(e):.3f}", flush=True)
