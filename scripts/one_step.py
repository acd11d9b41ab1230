"""The bench's C5 step (hsad_reduce + the four window-pair groups of fused detectors) run
`reps` times on the resident cube — for ncu captures of exactly one step's launches.

    python scripts/one_step.py [reps]
"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_1201_2025_b200 as hs  # noqa: E402
from harness.scene import CONFIGS, generate_rows  # noqa: E402
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"],
                     device="cuda")
reqs = bench.requests(hs)
st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
red = torch.empty((cfg["lines"], cfg["samples"], 4), dtype=torch.float64, device="cuda")
outs = None
for _ in range(reps):
    hs.reduce_detect(cube, reqs[:3], 2, 4, status=st, reduced=red)
    for g in range(1, 4):
        o = hs.detect_multi(red, reqs[3 * g:3 * g + 3], status=st)
torch.cuda.synchronize()
print("ok", int(st.item()))
