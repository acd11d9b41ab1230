"""DMMA reduction vs the oracle and vs the default kernel (HSAD_REDUCE_DMMA=1 set by caller)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1201_2025_b200 as hs, oracle
for bands, shape in ((224, (9, 13)), (64, (5, 30)), (224, (64, 100))):
    cube = oracle.port.random_cube(*shape, bands, bands).astype(np.float32)
    got = hs.reduce_cube(torch.as_tensor(cube).cuda(), 2, 4).cpu().numpy()
    want = oracle.port.reduce_cube(cube, 2, 4)
    print(bands, shape, "max rel", oracle.max_rel_diff(got, want))
