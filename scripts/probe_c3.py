"""Timing probe for the full-band path (BASELINE C3: 100x100x189, LRX 15 / guard 5)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_scene

cfg = CONFIGS["C3"]
cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"], device="cuda")
for label, req in [("lrx15", hs.DetectRequest("lrx", hs.WindowConfig.single(15))),
                   ("lrx15g5", hs.DetectRequest("lrx", hs.WindowConfig.single(15), guard=5))]:
    st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    outs = hs.detect_multi(cube, [req], status=st)
    for _ in range(2):
        hs.detect_multi(cube, [req], status=st, outputs=outs)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(5):
        hs.detect_multi(cube, [req], status=st, outputs=outs)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 5
    N = 224 if label == "lrx15" else 200
    L = 189
    flops = 1e4 * (N * L * (L + 1) + N * L + L ** 3 / 3 + L ** 2 + 2 * L)
    print(f"C3 {label}: {ms:.3f} ms  {1e4 / ms / 1e3:.2f} Mpix/s  {flops / ms / 1e9:.2f} TFLOP/s (alg)", flush=True)
