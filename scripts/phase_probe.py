"""Per-phase cycle breakdown of the fused detector (debug build with -DHSAD_PHASE_TIMERS)."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["HSAD_B200_LIB"] = str(Path(__file__).resolve().parents[1] / "paper_1201_2025_b200/libhsad_b200_pt.so")
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows
lib = hs._abi.lib()
lib.hsad_phase_cycles.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, 1024, cfg["rate"], device="cuda")
red = hs.reduce_cube(cube, 2, 4)
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
        hs.DetectRequest("dwest", W2(5, 11), eigcount=True)]
st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
hs.detect_multi(red, reqs, status=st); torch.cuda.synchronize()
buf = (C.c_ulonglong * 8)()
lib.hsad_phase_cycles(buf, 1)
hs.detect_multi(red, reqs, status=st); torch.cuda.synchronize()
lib.hsad_phase_cycles(buf, 1)
names = ["vertical update", "barrier A", "horizontal+centre", "solves (all)", "barrier B", "LRX->dual stats+DWRX", "DWEST"]
tot = sum(buf[i] for i in range(5))
for i, n in enumerate(names):
    print(f"{n:24s} {buf[i]/1e9:8.2f} Gcyc  {100*buf[i]/tot:5.1f}%")
