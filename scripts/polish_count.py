"""Debug build: average fp64 polish sweeps per warp-pixel-group in DWEST (C5 sweep windows)."""
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
rows = 512
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, rows, cfg["rate"], device="cuda")
red = hs.reduce_cube(cube, 2, 4)
W2 = hs.WindowConfig.dual
buf = (C.c_ulonglong * 8)()
for i, o in [(3, 7), (5, 11), (5, 15), (7, 21)]:
    lib.hsad_phase_cycles(buf, 1)
    hs.detect_multi(red, [hs.DetectRequest("dwest", W2(i, o))]); torch.cuda.synchronize()
    lib.hsad_phase_cycles(buf, 1)
    warps = rows * cfg["samples"] / 32
    print(f"{i}/{o}: polish sweeps per warp {buf[7] / warps:.3f}")
