"""Scratch timing probe: kernel times of reduce + fused detect on C4/C5 (CUDA events)."""
import sys, time
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
    ts.sort(); return ts[len(ts)//2]

for name in sys.argv[1:] or ["C4", "C5"]:
    cfg = CONFIGS[name]
    t0 = time.time()
    cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"], device="cuda")
    torch.cuda.synchronize(); print(name, "gen s", round(time.time()-t0, 2), flush=True)
    red = hs.reduce_cube(cube, 2, 4)
    npx = cfg["lines"] * cfg["samples"]
    tr = timeit(lambda: hs.reduce_cube(cube, 2, 4))
    gbs = npx * (cfg["bands"] * 4 + 32) / tr / 1e6
    print(f"{name} reduce ms {tr:.3f}  GB/s(alg in+out) {gbs:.0f}", flush=True)
    W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
    for label, reqs in [("lrx", [hs.DetectRequest("lrx", W1(11))]),
                        ("dwrx", [hs.DetectRequest("dwrx", W2(5, 11))]),
                        ("dwest", [hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]),
                        ("all3", [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
                                  hs.DetectRequest("dwest", W2(5, 11), eigcount=True)])]:
        st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        outs = hs.detect_multi(red, reqs, status=st)
        td = timeit(lambda: hs.detect_multi(red, reqs, status=st, outputs=outs))
        print(f"{name} detect {label} ms {td:.3f}  Mpix/s {npx/td/1e3:.0f}", flush=True)
    del cube, red; torch.cuda.empty_cache()
    if cfg["bands"] % 16 == 0:
        cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"], device="cuda")
        reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
                hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
        st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        red, outs = hs.reduce_detect(cube, reqs, status=st)
        tf = timeit(lambda: hs.reduce_detect(cube, reqs, status=st, reduced=red, outputs=outs))
        print(f"{name} FUSED reduce+detect all3 ms {tf:.3f}  Mpix/s {npx/tf/1e3:.0f}", flush=True)
        import os
        for env in ("HSAD_FUSED_DWT_ONLY", "HSAD_NO_FUSE"):
            os.environ[env] = "1"
            tf = timeit(lambda: hs.reduce_detect(cube, reqs, status=st, reduced=red, outputs=outs))
            print(f"{name} {env} ms {tf:.3f}", flush=True)
            del os.environ[env]
