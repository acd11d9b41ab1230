"""A/B probe: C5 sweep detector time with an env switch set / unset (argv[1] = env name)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows


def timeit(fn, n=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(n):
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); return ts[len(ts) // 2]


cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"], device="cuda")
red = hs.reduce_cube(cube, 2, 4)
del cube; torch.cuda.empty_cache()
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
env = sys.argv[1] if len(sys.argv) > 1 else None
for mode in ("on", "off"):
    if env and mode == "off":
        os.environ[env] = "1"
    tot, line = 0.0, []
    for inner, outer in [(3, 7), (5, 11), (5, 15), (7, 21)]:
        reqs = [hs.DetectRequest("lrx", W1(outer)), hs.DetectRequest("dwrx", W2(inner, outer)),
                hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)]
        st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        outs = hs.detect_multi(red, reqs, status=st)
        td = timeit(lambda: hs.detect_multi(red, reqs, status=st, outputs=outs))
        tot += td
        line.append(f"{inner}/{outer} {td:.3f}")
    print(f"{env}={'unset' if mode == 'on' else '1'}: " + "  ".join(line) + f"  sum {tot:.3f}", flush=True)
