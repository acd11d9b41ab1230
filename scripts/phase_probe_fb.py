"""Per-phase cycle breakdown of the full-band kernel on C3 (debug build, scripts/build_pt.sh)."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["HSAD_B200_LIB"] = str(Path(__file__).resolve().parents[1] / "paper_1201_2025_b200/libhsad_b200_pt.so")
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_scene
lib = hs._abi.lib()
lib.hsad_fb_phase_cycles.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
cfg = CONFIGS["C3"]
cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"], device="cuda")
reqs = [hs.DetectRequest("lrx", hs.WindowConfig.single(15), guard=5)]
buf = (C.c_ulonglong * 8)()
hs.detect_multi(cube, reqs); torch.cuda.synchronize()
lib.hsad_fb_phase_cycles(buf, 1)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); hs.detect_multi(cube, reqs); e.record(); torch.cuda.synchronize()
lib.hsad_fb_phase_cycles(buf, 1)
print("C3 ms", s.elapsed_time(e))
names = ["offsets+means", "centred Gram", "d+ridge", "Cholesky tail", "diag factor", "panels",
         "trailing update"]
tot = sum(buf[i] for i in range(7))
for i, n in enumerate(names):
    print(f"{n:16s} {buf[i]/1e6:10.1f} Mcyc  {100*buf[i]/tot:5.1f}%   per px {buf[i]/1e4:9.0f} cyc")
