"""How many C5 pixels the accuracy repair recomputes, and what it costs.

    python scripts/probe_repair.py
Runs the C5 sweep detectors with the repair on (default threshold) and off
(HSAD_NO_REPAIR=1 is read per call) and counts pixels whose scores differ."""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_1201_2025_b200 as hs  # noqa: E402
from harness.scene import CONFIGS, generate_rows  # noqa: E402

cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"],
                     device="cuda")
red = hs.reduce_cube(cube, 2, 4)
del cube
torch.cuda.empty_cache()
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
for inner, outer in [(3, 7), (5, 11), (5, 15), (7, 21)]:
    reqs = [hs.DetectRequest("lrx", W1(outer)), hs.DetectRequest("dwrx", W2(inner, outer)),
            hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)]
    res = {}
    for kappa in ("on", "off"):
        os.environ.pop("HSAD_NO_REPAIR", None) if kappa == "on" else os.environ.__setitem__("HSAD_NO_REPAIR", "1")
        st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        outs = hs.detect_multi(red, reqs, status=st)
        for _ in range(2):
            hs.detect_multi(red, reqs, status=st, outputs=outs)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        ts = []
        for _ in range(5):
            s.record(); hs.detect_multi(red, reqs, status=st, outputs=outs); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e))
        res[kappa] = (sorted(ts)[2], [o[0].clone() for o in outs])
    diff = [int((a != b).sum()) for a, b in zip(res["on"][1], res["off"][1])]
    print(f"{inner}/{outer}: repair on {res['on'][0]:.3f} ms, off {res['off'][0]:.3f} ms, "
          f"pixels changed by the repair lrx/dwrx/dwest {diff}", flush=True)
