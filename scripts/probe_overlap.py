"""C5 step: hsad_reduce of the whole cube then the four forked groups (the bench step) vs the
reduction in two row halves with each half's detector groups forked as soon as their reduced
rows exist (K1 of the second half runs next to the detectors of the first)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows

cfg = CONFIGS["C5"]
L, S, B = cfg["lines"], cfg["samples"], cfg["bands"]
cube = generate_rows(L, S, B, cfg["seed"], 0, L, cfg["rate"], device="cuda")
lib = hs._abi.lib()
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
SWEEP = [(7, 21), (5, 15), (5, 11), (3, 7)]
reqs = []
for i, o in SWEEP:
    reqs += [hs.DetectRequest("lrx", W1(o)), hs.DetectRequest("dwrx", W2(i, o)),
             hs.DetectRequest("dwest", W2(i, o), eigcount=True)]
st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
red = torch.empty((L, S, 4), dtype=torch.float64, device="cuda")
outs = [(torch.empty((L, S), dtype=torch.float64, device="cuda"),
         torch.empty((L, S), dtype=torch.int8, device="cuda") if r.eigcount else None) for r in reqs]
Req = hs._abi.Request
full = (Req * len(reqs))(*[hs.hsad._make_request(r, sc, cnt) for r, (sc, cnt) in zip(reqs, outs)])


def base():
    s = torch.cuda.current_stream().cuda_stream
    assert lib.hsad_reduce_detect(cube.data_ptr(), L, S, B, 2, 4, 0, L, 0, L, red.data_ptr(), full, len(reqs),
                                  st.data_ptr(), None, s) == 0


def halves(nparts):
    # parts of rows; part p's detectors need reduced rows up to its end + 10 (+ quantum slack)
    main = torch.cuda.current_stream()
    q = 32
    bounds = [round(L * p / nparts / q) * q for p in range(nparts + 1)]
    halo = 32
    done_to = 0
    for p in range(nparts):
        r0, r1 = bounds[p], bounds[p + 1]
        need = min(L, r1 + halo)
        if need > done_to:
            assert lib.hsad_reduce(cube[done_to:need].data_ptr(), 4, need - done_to, S, B, 2, 4,
                                   red[done_to:need].data_ptr(), 8, main.cuda_stream) == 0
            done_to = need
        sub = (Req * len(reqs))(*[hs.hsad._make_request(r, sc[r0:r1], None if cnt is None else cnt[r0:r1])
                                  for r, (sc, cnt) in zip(reqs, outs)])
        keep.append(sub)
        side = sides[p % len(sides)]
        side.wait_stream(main)
        with torch.cuda.stream(side):
            assert lib.hsad_detect_multi(red.data_ptr(), 8, L, S, 4, 0, L, r0, r1, sub, len(reqs), st.data_ptr(),
                                         None, side.cuda_stream) == 0
    for side in sides:
        main.wait_stream(side)


keep = []
sides = [torch.cuda.Stream() for _ in range(4)]


def timeit(fn, n=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
        keep.clear()
    ts.sort()
    return ts[len(ts) // 2]


print(f"one reduce + forked groups   {timeit(base):.3f} ms")
ref = [o[0].clone() for o in outs]
for n in (2, 4, 8):
    print(f"{n} row parts, pipelined       {timeit(lambda: halves(n)):.3f} ms  bit-identical: "
          f"{all(torch.equal(a, o[0]) for a, o in zip(ref, outs))}")
print(f"one reduce + forked groups   {timeit(base):.3f} ms")
