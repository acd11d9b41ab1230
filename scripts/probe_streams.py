"""C5 sweep detectors: the four window-pair launches back to back on one stream vs forked onto
four streams (their inputs are the same reduced cube; they do not depend on each other)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows

cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"], device="cuda")
red = hs.reduce_cube(cube, 2, 4)
del cube
torch.cuda.empty_cache()
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
SWEEP = [(3, 7), (5, 11), (5, 15), (7, 21)]
groups = [[hs.DetectRequest("lrx", W1(o)), hs.DetectRequest("dwrx", W2(i, o)),
           hs.DetectRequest("dwest", W2(i, o), eigcount=True)] for i, o in SWEEP]
sts = [torch.full((1,), -1, dtype=torch.int64, device="cuda") for _ in groups]
outs = [hs.detect_multi(red, g, status=st) for g, st in zip(groups, sts)]
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in groups]


def seq():
    for g, st, o in zip(groups, sts, outs):
        hs.detect_multi(red, g, status=st, outputs=o)


def fork(order=(0, 1, 2, 3)):
    main = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(main)
    for k in order:
        s = streams[k]
        s.wait_event(ev)
        with torch.cuda.stream(s):
            hs.detect_multi(red, groups[k], status=sts[k], outputs=outs[k])
    for s in streams:
        main.wait_stream(s)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


print(f"sequential {timeit(seq):.3f} ms")
print(f"forked     {timeit(fork):.3f} ms")
print(f"forked rev {timeit(lambda: fork((3, 2, 1, 0))):.3f} ms")
print(f"sequential {timeit(seq):.3f} ms")
