"""Probe: end to end from raw ENVI bytes on the host (hsad_pipeline_raw) for the C5 sweep:
int16 BSQ (7.5 GB, the AVIRIS on-disk type) and fp32 BSQ (15 GB), vs a bare pinned H2D."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1201_2025_b200 as hs
from paper_1201_2025_b200 import evalio
import bench

L, S, B = 4096, 4096, 224
reqs = bench.requests(hs)
outs = [(torch.empty((L, S), dtype=torch.float64, pin_memory=True),
         torch.empty((L, S), dtype=torch.int8, pin_memory=True) if r.eigcount else None) for r in reqs]
for code, dt in ((2, torch.int16), (4, torch.float32)):
    host = torch.empty(L * S * B, dtype=dt, pin_memory=True)
    g = torch.Generator().manual_seed(5)
    if dt == torch.int16:
        host.copy_(torch.randint(0, 4000, (L * S * B,), dtype=torch.int16, generator=g))
    else:
        host.normal_(generator=g)
    raw = host.view(torch.uint8)
    hdr = evalio.CubeHeader(S, L, B, "bsq", code, 0)
    evalio.pipeline_raw(raw, hdr, 2, 4, reqs, outs)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); evalio.pipeline_raw(raw, hdr, 2, 4, reqs, outs); ts.append(time.perf_counter() - t0)
    dev = torch.empty_like(host, device="cuda")
    torch.cuda.synchronize(); t1 = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize()
    h2d = time.perf_counter() - t1
    e2e = sorted(ts)[1]
    print(f"BSQ code {code}: e2e {e2e*1e3:.1f} ms = {L*S/e2e/1e6:.1f} Mpix/s; bare H2D {h2d*1e3:.1f} ms "
          f"({raw.numel()/h2d/1e9:.1f} GB/s)", flush=True)
    del host, dev, raw
