"""Run each hot kernel a few times on a rows x 4096 x 224 slice of the C5 scene (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1201_2025_b200 as hs  # noqa: E402
from harness.scene import CONFIGS, generate_rows  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, rows, cfg["rate"],
                     device="cuda")
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
        hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
lrx_only = [reqs[0]]
st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
for _ in range(3):
    red = hs.reduce_cube(cube, 2, 4)
    outs = hs.detect_multi(red, reqs, status=st)
    hs.detect_multi(red, lrx_only, status=st)
torch.cuda.synchronize()
print("ok", int(st.item()))
