"""Probe: distribution of DWEST eigen-counts on the C5 sweep (per pixel and per warp of 32 columns)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows

cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, 1024, cfg["rate"], device="cuda")
red = hs.reduce_cube(cube, 2, 4)
for inner, outer in [(3, 7), (5, 11), (5, 15), (7, 21)]:
    (s, c), = hs.detect_multi(red, [hs.DetectRequest("dwest", hs.WindowConfig.dual(inner, outer), eigcount=True)])
    c = c.to(torch.int64)
    hist = torch.bincount(c.flatten(), minlength=5)[:5].tolist()
    w = c.view(c.shape[0], -1, 32).amax(dim=2)
    whist = torch.bincount(w.flatten(), minlength=5)[:5].tolist()
    print(f"{inner}/{outer} pixel counts {hist}  warp-max counts {whist}", flush=True)
