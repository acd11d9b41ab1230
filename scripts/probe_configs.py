"""Probe: every BASELINE config (C1-C4; C5 is bench.py) on one B200 — device-resident time,
end-to-end time through hsad_pipeline_host (pinned host cube in, host maps out), the CPU
oracle on all host cores for the same job, and the parity gates (max rel diff vs the oracle,
identical DWEST eigen-counts, identical top-k sets with k = truth positives).

    python scripts/probe_configs.py > profiles/configs_r2.json
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import oracle
import paper_1201_2025_b200 as hs
from paper_1201_2025_b200 import evalio
from harness.scene import CONFIGS, generate_scene

W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
JOBS = {
    "C1": (2, [("lrx", W1(9), 3)]),
    "C2": (2, [("dwrx", W2(5, 11), 1), ("dwest", W2(5, 11), 1)]),
    "C3": (0, [("lrx", W1(15), 5)]),
    "C4": (2, [("lrx", W1(11), 1), ("dwrx", W2(5, 11), 1), ("dwest", W2(5, 11), 1)]),
}
cores = os.cpu_count() or 1


def reqs_of(spec):
    return [hs.DetectRequest(a, w, guard=g, eigcount=(a == "dwest")) for a, w, g in spec]


def oracle_maps(cube, order, spec):
    red = oracle.port.reduce_cube(cube, order, 4, workers=cores) if order else cube
    out = []
    for a, w, g in spec:
        if a == "lrx":
            out.append((oracle.port.local_rx(red, w.single_size, 1e-6, guard=g, workers=cores), None))
        elif a == "dwrx":
            out.append((oracle.port.dwrx(red, w.inner_size, w.outer_size, 1e-6, workers=cores), None))
        else:
            out.append(oracle.port.dwest(red, w.inner_size, w.outer_size, 0.1, workers=cores))
    return out


def topk_set(scores, k):
    order = np.lexsort((np.arange(scores.size), -scores.ravel()))
    return set(order[:k].tolist())


result = {"cores": cores, "gpu": torch.cuda.get_device_name(0), "configs": {}}
for name, (order, spec) in JOBS.items():
    cfg = CONFIGS[name]
    cube, truth = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"],
                                 device="cuda")
    reqs = reqs_of(spec)
    lines, samples = cfg["lines"], cfg["samples"]

    def device_run():
        src = hs.reduce_cube(cube, order, 4) if order else cube
        return hs.detect_multi(src, reqs)

    outs = device_run()
    torch.cuda.synchronize()
    # device time: the C-ABI calls (async status, preallocated outputs) captured once in
    # a CUDA graph and replayed, so host-side launch overhead does not count
    st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    red = hs.reduce_cube(cube, order, 4) if order else cube
    lib = hs._abi.lib()
    g_reqs = (hs._abi.Request * len(reqs))(*[hs.hsad._make_request(r, sc, cnt)
                                              for r, (sc, cnt) in zip(reqs, outs)])
    bands = cfg["bands"]

    def capture_body():
        strm = torch.cuda.current_stream().cuda_stream
        if order:
            assert lib.hsad_reduce(cube.data_ptr(), cube.element_size(), lines, samples, bands, order, 4,
                                   red.data_ptr(), 8, strm) == 0
        src = red if order else cube
        assert lib.hsad_detect_multi(src.data_ptr(), src.element_size(), lines, samples,
                                     4 if order else bands, 0, lines, 0, lines, g_reqs, len(reqs),
                                     st.data_ptr(), None, strm) == 0

    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        capture_body()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        capture_body()
    ts = []
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for _ in range(20):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); graph.replay(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    dev_ms = statistics.median(ts)
    assert int(st.item()) == -1
    # end to end from pinned host memory
    hcube = cube.float().cpu().pin_memory()
    hout = [(torch.empty((lines, samples), dtype=torch.float64).pin_memory(),
             torch.empty((lines, samples), dtype=torch.int8).pin_memory() if r.eigcount else None)
            for r in reqs]
    hs.pipeline_host(hcube, order, 4, reqs, hout)
    te = []
    for _ in range(5):
        t0 = time.perf_counter(); hs.pipeline_host(hcube, order, 4, reqs, hout); te.append(time.perf_counter() - t0)
    e2e_ms = statistics.median(te) * 1e3
    # CPU oracle (all cores) on the same bytes
    cube_np = cube.double().cpu().numpy() if order == 0 else cube.float().cpu().numpy().astype(np.float64)
    t0 = time.perf_counter()
    want = oracle_maps(cube_np, order, spec)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    # parity gates
    k = int(truth.sum().item())
    gates = []
    for (a, w, g), (sc, cnt), (ws, wc) in zip(spec, outs, want):
        got = sc.cpu().numpy()
        err = oracle.max_rel_diff(got, ws)
        idx, _ = evalio.top_k(sc, k)
        gates.append({"detector": a, "window": w.describe() + (f" guard {g}" if g > 1 else ""),
                      "max_rel_diff": err,
                      "topk_identical": set(idx.cpu().numpy().tolist()) == topk_set(ws, k),
                      "eigcount_identical": None if wc is None else bool(np.array_equal(cnt.cpu().numpy(), wc))})
    px = lines * samples
    result["configs"][name] = {
        "shape": [lines, samples, cfg["bands"]], "dwt": bool(order), "k": k,
        "device_ms": dev_ms, "device_mpix_s": px / dev_ms / 1e3,
        "e2e_ms": e2e_ms, "e2e_mpix_s": px / e2e_ms / 1e3,
        "cpu_oracle_ms": cpu_ms, "cpu_oracle_mpix_s": px / cpu_ms / 1e3,
        "speedup_e2e_vs_cpu": cpu_ms / e2e_ms, "gates": gates}
    print(name, json.dumps(result["configs"][name]), file=sys.stderr, flush=True)
print(json.dumps(result, indent=1))
