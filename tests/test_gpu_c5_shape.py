"""Parity at the benchmarked launch shape (BASELINE configs[4], the C5 sweep).

C5 (4096 x 4096 x 224 fp32) runs the detectors with the full-size row quantum (the
longest fp64 running-sum chains after the window warm-up) on 4096-column strips and
the 4-pair window sweep 7/3, 11/5, 15/5, 21/7. Smaller test images get a smaller
quantum (the grid must still fill the GPU), so this test picks the smallest image
height at 4096 columns whose quantum equals C5's, generates it with the BASELINE
generator (harness/scene_gen.cpp, C5 seed and anomaly rate), runs the benchmark's
exact request list through the C-ABI, and checks SURVEY 8d's deterministic row subset
(top border + first chunk, shard boundaries +-R for G in {2,4,8}, chunk ends, seeded
random rows, bottom border) against the oracle: fp64 maps <= 1e-9 (rel_diff of
proj/tests/support/testutil.hpp:34-36), DWT <= 1e-5, identical DWEST eigen-counts and
top-k sets. The reference pattern is proj/tests/acceptance/acceptance_main.cpp:190-208
(detectors vs the naive oracle on a seeded cube). The host pipeline
(hsad_pipeline_host, row strips from pinned memory) must reproduce the device maps
bit for bit.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_1201_2025_b200")
import bench  # noqa: E402
from harness.scene import CONFIGS, anomaly_fill, generate_rows  # noqa: E402

DEV = "cuda:0"


def c5_shape_lines(samples=4096):
    q5 = hs.row_quantum(4096, samples)
    lines = q5
    while hs.row_quantum(lines, samples) != q5:
        lines += q5
    return lines, q5


def test_c5_launch_shape_sweep_matches_oracle(orc):
    cfg = CONFIGS["C5"]
    samples, bands = cfg["samples"], cfg["bands"]
    lines, q = c5_shape_lines(samples)
    assert q == hs.row_quantum(cfg["lines"], samples) and q >= 32
    host_cube = generate_rows(lines, samples, bands, cfg["seed"], 0, lines, cfg["rate"], pin=True)
    cube = host_cube.to(DEV)
    reqs = bench.requests(hs)
    red = hs.reduce_cube(cube, 2, 4)
    del cube
    outs = hs.detect_multi(red, reqs)
    torch.cuda.synchronize()

    rows = bench.parity_rows(lines, q, n_random=32, seed=0xC5)
    idx = torch.tensor(rows, device=DEV)
    maps = [lambda r, sc=sc, cnt=cnt: (sc[idx].cpu().numpy(),
                                       None if cnt is None else cnt[idx].cpu().numpy())
            for sc, cnt in outs]
    truth, _ = anomaly_fill(lines, samples, cfg["rate"], cfg["seed"])
    par = bench.oracle_parity(host_cube.numpy(), lines, rows, lambda a, b: red[a:b].cpu().numpy(),
                              maps, truth[rows], os.cpu_count() or 1)
    assert par["dwt_max_rel_diff"] <= 1e-5, par
    assert max(par["max_rel_diff"].values()) <= 1e-9, par["max_rel_diff"]
    assert not any(par["eigcount_mismatches"]), par["eigcount_mismatches"]
    assert all(par["topk_identical"]), par
    assert par["pass"]

    # end to end from pinned host memory: bit-identical to the device-resident maps
    host_out = [(torch.empty((lines, samples), dtype=torch.float64, pin_memory=True),
                 torch.empty((lines, samples), dtype=torch.int8, pin_memory=True)
                 if r.eigcount else None) for r in reqs]
    hs.pipeline_host(host_cube, 2, 4, reqs, host_out)
    torch.cuda.synchronize()
    for (sc, cnt), (hsc, hcnt) in zip(outs, host_out):
        assert torch.equal(sc.cpu(), hsc)
        if cnt is not None:
            assert torch.equal(cnt.cpu(), hcnt)
