"""Small end-to-end exercise of every kernel for compute-sanitizer (memcheck)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1201_2025_b200 as hs
import oracle

dev = "cuda:0"
W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
for shape, bands in (((23, 31), 4), ((6, 9), 4), ((40, 5), 3), ((130, 300), 4), ((7, 7), 8),
                     ((70, 129), 4), ((33, 2100), 4)):
    cube = torch.as_tensor(oracle.port.random_cube(*shape, bands, 7)).to(dev)
    reqs = [hs.DetectRequest("lrx", W1(11)), hs.DetectRequest("dwrx", W2(5, 11)),
            hs.DetectRequest("dwest", W2(5, 11), eigcount=True), hs.DetectRequest("lrx", W1(9), guard=3)]
    hs.detect_multi(cube, reqs)
    hs.detect_multi(cube, reqs[:3])  # standard layout: the TMA-staged kernel
    hs.detect_multi(cube.float(), reqs[:2])
full = torch.as_tensor(oracle.port.random_cube(37, 45, 189, 9)).to(dev)
for out_dtype in (torch.float64, torch.float32):
    hs.reduce_cube(full, 2, 4, out_dtype=out_dtype)
hs.reduce_cube(full.float(), 2, 8)
hs.reduce_cube(full, 2, 16)
red = hs.reduce_cube(full.float(), 2, 4)
q = hs.row_quantum(37, 45)
b0, nb = hs.strip_rows(37, q, 2 * q, reqs)
hs.detect_multi(red[b0:b0 + nb].contiguous(), reqs, lines=37, buf_row0=b0, row_begin=q, row_end=2 * q)
fb = torch.as_tensor(oracle.port.random_cube(9, 11, 30, 3)).to(dev)
hs.detect_multi(fb, [hs.DetectRequest("lrx", W1(7)), hs.DetectRequest("dwrx", W2(3, 7))])
flat = torch.zeros((5, 5, 2), dtype=torch.float64, device=dev); flat[2, 2] = 1.0
try:
    hs.local_rx(flat, W1(3))
except hs.HsadError:
    pass
torch.cuda.synchronize()
print("sanitize ok")
