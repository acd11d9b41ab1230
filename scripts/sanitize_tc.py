"""Small exercise of the tcgen05 window-Gram route (HSAD_FB_TC=1) for compute-sanitizer (memcheck)."""
import os
import sys
from pathlib import Path
os.environ["HSAD_FB_TC"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
import oracle

dev = "cuda:0"
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
for shape, bands, w, inner in (((9, 11), 30, 7, 3), ((12, 60), 189, 9, 3), ((5, 7), 120, 5, 3), ((14, 53), 64, 11, 5)):
    fb = torch.as_tensor(oracle.port.random_cube(*shape, bands, 3)).to(dev)
    hs.detect_multi(fb, [hs.DetectRequest("lrx", W1(w)), hs.DetectRequest("dwrx", W2(inner, w)),
                         hs.DetectRequest("lrx", W1(w), guard=3)])
    hs.detect_multi(fb.double(), [hs.DetectRequest("lrx", W1(w))])
torch.cuda.synchronize()
print("sanitize tc ok")
