"""C3 full-band DWEST (100x100x189 raw cube, 5/15 windows): device time and eigen-counts.

    python scripts/probe_c3_dwest.py [out.json]
"""
import json
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1201_2025_b200 as hs  # noqa: E402
from harness.scene import CONFIGS, generate_scene  # noqa: E402

cfg = CONFIGS["C3"]
cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"], device="cuda")
reqs = [hs.DetectRequest("dwest", hs.WindowConfig.dual(5, 15), eigcount=True)]
st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
outs = hs.detect_multi(cube, reqs, status=st)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
ts = []
for _ in range(5):
    s.record(); hs.detect_multi(cube, reqs, status=st, outputs=outs); e.record(); e.synchronize()
    ts.append(s.elapsed_time(e))
cnt = outs[0][1].cpu().numpy()
res = {"config": "C3 100x100x189 raw, DWEST 5/15 full band", "ms": sorted(ts)[2],
       "us_per_pixel_per_sm": sorted(ts)[2] * 1e3 * 148 / 1e4,
       "eigcount_hist": np.bincount(cnt.ravel()).tolist(), "status": int(st.item())}
print(json.dumps(res))
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(res, indent=1))
