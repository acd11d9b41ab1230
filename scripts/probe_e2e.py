"""Probe: C5 end-to-end (hsad_pipeline_host, 12 maps) vs a bare pinned H2D of the cube.
HSAD_B200_LIB selects the library build."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from harness.scene import CONFIGS, generate_rows
import bench

cfg = CONFIGS["C5"]
cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"], cfg["rate"], device="cuda")
host = torch.empty(cube.shape, dtype=torch.float32, pin_memory=True)
host.copy_(cube)
del cube
torch.cuda.empty_cache()
reqs = bench.requests(hs)
L, S = cfg["lines"], cfg["samples"]
outs = [(torch.empty((L, S), dtype=torch.float64, pin_memory=True),
         torch.empty((L, S), dtype=torch.int8, pin_memory=True) if r.eigcount else None) for r in reqs]
hs.pipeline_host(host, 2, 4, reqs, outs)
torch.cuda.synchronize()
dev = torch.empty_like(host, device="cuda")
for rep in range(3):
    t0 = time.perf_counter(); hs.pipeline_host(host, 2, 4, reqs, outs); e2e = time.perf_counter() - t0
    torch.cuda.synchronize()
    t1 = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t1
    print(f"{Path(os.environ.get('HSAD_B200_LIB', 'default')).name}: e2e {e2e*1e3:.1f} ms  bare H2D {h2d*1e3:.1f} ms", flush=True)
