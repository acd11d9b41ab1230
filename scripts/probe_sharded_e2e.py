"""C5 end to end from pinned host memory: hsad_pipeline_host vs hsad_pipeline_sharded
(n_strips 1 / 8) on the visible GPUs; wall times and map bit-identity.

    python scripts/probe_sharded_e2e.py [out.json]
"""
import json
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_1201_2025_b200 as hs  # noqa: E402
from paper_1201_2025_b200.sharded import pipeline_sharded  # noqa: E402
from harness.scene import CONFIGS, generate_rows  # noqa: E402
import bench  # noqa: E402

cfg = CONFIGS["C5"]
L, S, B = cfg["lines"], cfg["samples"], cfg["bands"]
h = generate_rows(L, S, B, cfg["seed"], 0, L, cfg["rate"], pin=True)
reqs = bench.requests(hs)


def outs():
    return [(torch.empty((L, S), dtype=torch.float64, pin_memory=True),
             torch.empty((L, S), dtype=torch.int8, pin_memory=True) if r.eigcount else None) for r in reqs]


res = {"devices": torch.cuda.device_count()}
ref = outs()
hs.pipeline_host(h, 2, 4, reqs, ref)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); hs.pipeline_host(h, 2, 4, reqs, ref); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
res["pipeline_host_ms"] = min(ts) * 1e3
for n in (1, 8):
    o = outs()
    pipeline_sharded(h, 2, 4, reqs, o, n)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); pipeline_sharded(h, 2, 4, reqs, o, n); ts.append(time.perf_counter() - t0)
    same = all(torch.equal(a, b) and (ac is None or torch.equal(ac, bc)) for (a, ac), (b, bc) in zip(o, ref))
    res[f"pipeline_sharded_{n}_ms"] = min(ts) * 1e3
    res[f"pipeline_sharded_{n}_bit_identical"] = same
print(json.dumps(res), flush=True)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(res, indent=1))
