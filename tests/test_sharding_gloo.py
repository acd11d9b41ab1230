"""Multi-rank path on CPU: world_size 2 (and 3) with the gloo backend.

Each rank plans its row strip, takes only its buffer rows (strip + mirror halo) from
the host copy, computes them — here with the CPU oracle standing in for the CUDA
kernels, since this box has no GPU — and the maps are gathered to rank 0. Rows
outside a rank's buffer are NaN-poisoned, so a wrong halo shows up as NaN scores.
The gathered maps must equal the single-process oracle maps exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LINES, SAMPLES, BANDS = 37, 23, 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_compute(full_cube):
    """Per-strip compute with the oracle: sees only the buffer rows of the strip."""
    import oracle

    def compute(buf, plan, requests, order, target):
        lines = plan.lines
        poisoned = np.full((lines,) + tuple(buf.shape[1:]), np.nan, np.float64)
        poisoned[plan.b0: plan.b0 + plan.nb] = buf.numpy()
        # the oracle reduces every row; rows outside the buffer stay NaN
        red = np.full((lines, buf.shape[1], target), np.nan)
        red[plan.b0: plan.b0 + plan.nb] = oracle.port.reduce_cube(buf.numpy(), order, target)
        outs = []
        for r in requests:
            rows = (plan.r0, plan.r1)
            if r.algorithm == "lrx":
                s = oracle.port.local_rx(red, r.window.single_size, r.ridge, rows=rows)
                outs.append((torch.from_numpy(s), None))
            elif r.algorithm == "dwrx":
                s = oracle.port.dwrx(red, r.window.inner_size, r.window.outer_size, r.ridge, rows=rows)
                outs.append((torch.from_numpy(s), None))
            else:
                s, c = oracle.port.dwest(red, r.window.inner_size, r.window.outer_size,
                                         r.eigen_fraction, rows=rows)
                outs.append((torch.from_numpy(s), torch.from_numpy(c)))
        return outs

    return compute


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1201_2025_b200 import DetectRequest, WindowConfig
        from paper_1201_2025_b200.sharded import run_sharded
        cube = oracle.port.random_cube(LINES, SAMPLES, BANDS, 4242)
        reqs = [DetectRequest("lrx", WindowConfig.single(7)),
                DetectRequest("dwrx", WindowConfig.dual(3, 9)),
                DetectRequest("dwest", WindowConfig.dual(3, 9), eigcount=True)]
        plan, maps, counts = run_sharded(
            lambda b0, b1: torch.from_numpy(cube[b0:b1].copy()), LINES, SAMPLES, reqs, dist,
            compute=_oracle_compute(cube))
        if rank == 0:
            q.put(("maps", [m.numpy() for m in maps], counts[2].numpy(), plan.per))
        q.put(("plan", rank, plan.r0, plan.r1, plan.b0, plan.nb))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_equals_single_process(orc, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    got = {}
    plans = []
    while not q.empty():
        item = q.get()
        if item[0] == "maps":
            got = item
        else:
            plans.append(item[1:])
    _, maps, counts, per = got
    cube = orc.port.random_cube(LINES, SAMPLES, BANDS, 4242)
    red = orc.port.reduce_cube(cube, 2, 4)
    want = [orc.port.local_rx(red, 7), orc.port.dwrx(red, 3, 9)]
    ds, dc = orc.port.dwest(red, 3, 9)
    want.append(ds)
    for m, w in zip(maps, want):
        assert np.all(np.isfinite(m)), "a rank read outside its halo"
        assert np.array_equal(m, w)
    assert np.array_equal(counts, dc)
    # strips tile the image; buffers are strip + halo within the image
    plans.sort()
    assert plans[0][1] == 0 and plans[-1][2] == LINES
    for (_, r0, r1, b0, nb) in plans:
        if r1 > r0:
            assert b0 <= max(0, r0 - 4) and b0 + nb >= min(LINES, r1 + 4)


def _grouped_worker(rank, world, port, q):
    """bench.py's N > 1 step: per window-pair group, the strip maps are written into
    padded (per, samples) buffers and gathered asynchronously (sharded.MapGather)
    while the next group computes; one wait at the end of the step."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1201_2025_b200 import DetectRequest, WindowConfig
        from paper_1201_2025_b200.sharded import MapGather, plan_strip
        cube = oracle.port.random_cube(LINES, SAMPLES, BANDS, 777)
        sweep = [(3, 7), (5, 11)]
        reqs = []
        for i, o in sweep:
            reqs += [DetectRequest("lrx", WindowConfig.single(o)),
                     DetectRequest("dwest", WindowConfig.dual(i, o), eigcount=True)]
        plan = plan_strip(LINES, SAMPLES, world, rank, reqs)
        g = MapGather(plan, dist)
        red = oracle.port.reduce_cube(cube, 2, 4)
        rows = (plan.r0, plan.r1)
        bufs = [(g.padded(torch.float64, "cpu"), g.padded(torch.int8, "cpu") if r.eigcount else None)
                for r in reqs]
        for step in range(2):  # receive buffers are reused across steps
            for gi, (i, o) in enumerate(sweep):
                s = oracle.port.local_rx(red, o, rows=rows)
                bufs[2 * gi][0][: plan.r1 - plan.r0].copy_(torch.from_numpy(s))
                ds, dc = oracle.port.dwest(red, i, o, rows=rows)
                bufs[2 * gi + 1][0][: plan.r1 - plan.r0].copy_(torch.from_numpy(ds))
                bufs[2 * gi + 1][1][: plan.r1 - plan.r0].copy_(torch.from_numpy(dc))
                for k in (2 * gi, 2 * gi + 1):
                    g.launch(2 * k, bufs[k][0])
                    if bufs[k][1] is not None:
                        g.launch(2 * k + 1, bufs[k][1])
            g.wait()
        if rank == 0:
            q.put([g.full(2 * k).numpy().copy() for k in range(len(reqs))] +
                  [g.full(3).numpy().copy(), g.full(7).numpy().copy()])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_grouped_async_gather_like_bench(orc, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grouped_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    got = q.get()
    cube = orc.port.random_cube(LINES, SAMPLES, BANDS, 777)
    red = orc.port.reduce_cube(cube, 2, 4)
    want = []
    counts = []
    for i, o in [(3, 7), (5, 11)]:
        want.append(orc.port.local_rx(red, o))
        s, c = orc.port.dwest(red, i, o)
        want.append(s)
        counts.append(c)
    for m, w in zip(got[:4], want):
        assert np.array_equal(m, w)
    assert np.array_equal(got[4], counts[0]) and np.array_equal(got[5], counts[1])


def test_strip_plan_tiles_the_image():
    """hsad_strip_plan (the split hsad_gather_maps, hsad_pipeline_sharded and the bench
    use): strips are contiguous, quantum-aligned and tile [0, lines) for any world size."""
    from paper_1201_2025_b200.hsad import row_quantum
    from paper_1201_2025_b200.sharded import plan_strip
    for lines, samples in ((4096, 4096), (512, 614), (37, 23), (100, 100), (5, 7)):
        q = row_quantum(lines, samples)
        for world in (1, 2, 3, 4, 8):
            plans = [plan_strip(lines, samples, world, r, []) for r in range(world)]
            assert plans[0].r0 == 0 and plans[-1].r1 == lines
            for a, b in zip(plans, plans[1:]):
                assert a.r1 == b.r0
            assert all(p.r0 % q == 0 and p.per % q == 0 for p in plans if p.r1 > p.r0)
