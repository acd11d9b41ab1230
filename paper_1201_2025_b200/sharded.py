"""Row-strip sharding of the hot path over the GPUs of one node.

The image splits into row strips whose boundaries are multiples of
hsad_row_quantum(lines, samples) — the chunk height the detector grid is anchored
to — so every pixel's arithmetic (tile shift, running-sum start) is the same at
any strip count and the 1/2/4/8-GPU score maps are bit-identical (the analogue of
the reference's worker-count invariance, proj/core/src/parallel.hpp:12-16).

Rank g owns output rows [r0, r1) and holds the full-band rows the windows of
those rows touch, [b0, b0 + nb) (hsad_strip_rows: outer-window radius halo with
the reference's reflection at the image edges, detect.cpp:71-76), taken from the
host copy. No data crosses ranks during compute; the only collective is the final
gather of the score maps to rank 0 (NCCL has no gather primitive: torch's
dist.gather issues the grouped sends/receives), on padded equal-size strips.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch

from .hsad import DetectRequest, detect_multi, reduce_cube, row_quantum, strip_rows


@dataclass(frozen=True)
class StripPlan:
    lines: int
    samples: int
    world: int
    rank: int
    quantum: int
    per: int      # padded rows per rank (multiple of quantum)
    r0: int       # output rows [r0, r1)
    r1: int
    b0: int       # buffer rows [b0, b0 + nb)
    nb: int


def plan_strip(lines: int, samples: int, world: int, rank: int,
               requests: Sequence[DetectRequest]) -> StripPlan:
    """The C-ABI's strip plan (hsad_strip_plan, the split hsad_gather_maps and
    hsad_pipeline_sharded use) plus the strip's buffer rows (hsad_strip_rows)."""
    import ctypes as C
    from . import _abi
    from .hsad import _check
    r0, r1, per = C.c_int64(), C.c_int64(), C.c_int64()
    _check(_abi.lib().hsad_strip_plan(lines, samples, world, rank, C.byref(r0), C.byref(r1),
                                      C.byref(per)))
    r0, r1 = r0.value, r1.value
    b0, nb = strip_rows(lines, r0, r1, requests) if r1 > r0 else (r0, 0)
    return StripPlan(lines, samples, world, rank, row_quantum(lines, samples), per.value, r0, r1,
                     b0, nb)


class NcclMapGather:
    """Score-map gather to rank `dst` through the C-ABI (hsad_gather_maps: grouped
    ncclSend / ncclRecv straight into the root's full maps) on an NCCL communicator the
    library creates from a unique id broadcast over `dist` (any backend).

    launch(slot, strip) enqueues one map's gather on the current stream; full(slot) is the
    root's (lines, samples) map, allocated once per slot and reused across calls."""

    def __init__(self, plan: StripPlan, dist, dst: int = 0):
        import ctypes as C
        from . import _abi
        from .hsad import _check
        self.plan, self.dst, self._C, self._abi = plan, dst, C, _abi
        self.full_maps: dict[int, torch.Tensor] = {}
        self.stream = None
        self.comm = C.c_void_p()
        if plan.world > 1:
            uid = (C.c_uint8 * 128)()
            if plan.rank == 0:
                _check(_abi.lib().hsad_nccl_unique_id(uid))
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend() == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0)
            uid = (C.c_uint8 * 128)(*t.cpu().tolist())
            _check(_abi.lib().hsad_nccl_comm_init_rank(C.byref(self.comm), plan.world, uid, plan.rank))

    def launch(self, slot: int, strip: torch.Tensor) -> None:
        """Enqueues the gather of `strip` on the gather stream once the current stream's
        work so far (the kernels that wrote it) is done: it overlaps the next kernels."""
        from .hsad import _check
        p = self.plan
        if self.stream is None:
            self.stream = torch.cuda.Stream(device=strip.device)
        self.stream.wait_stream(torch.cuda.current_stream(strip.device))
        full = None
        if p.rank == self.dst:
            full = self.full_maps.get(slot)
            if full is None:
                full = torch.empty((p.lines, p.samples), dtype=strip.dtype, device=strip.device)
                self.full_maps[slot] = full
        desc = (self._abi.MapDesc * 1)(self._abi.MapDesc(
            strip.data_ptr(), full.data_ptr() if full is not None else None, strip.element_size()))
        _check(self._abi.lib().hsad_gather_maps(self.comm, p.world, p.rank, self.dst, p.lines,
                                                p.samples, desc, 1, self.stream.cuda_stream))

    def wait(self) -> None:
        """The current stream waits for every gather launched so far."""
        if self.stream is not None:
            torch.cuda.current_stream(self.stream.device).wait_stream(self.stream)

    def full(self, slot: int) -> torch.Tensor | None:
        return self.full_maps.get(slot) if self.plan.rank == self.dst else None

    def close(self) -> None:
        if self.comm.value:
            self._abi.lib().hsad_nccl_comm_destroy(self.comm)
            self.comm = self._C.c_void_p()


def compute_strip_gpu(buf: torch.Tensor, plan: StripPlan, requests: Sequence[DetectRequest],
                      order: int = 2, target_bands: int = 4, status: torch.Tensor | None = None):
    """DWT of the strip's buffer rows, then the fused detectors on rows [r0, r1)."""
    if plan.r1 <= plan.r0:
        return [(torch.empty((0, plan.samples), dtype=r.score_dtype, device=buf.device), None)
                for r in requests]
    red = reduce_cube(buf, order, target_bands) if order > 0 else buf
    return detect_multi(red, requests, lines=plan.lines, buf_row0=plan.b0,
                        row_begin=plan.r0, row_end=plan.r1, status=status)


class MapGather:
    """Gathers padded (per, samples) strip maps to rank `dst`, one asynchronous
    dist.gather per map, so a group's maps travel while the next group of detectors
    still computes (NCCL: the collective stream waits on the compute stream at launch,
    the compute stream is free to run the next kernels; `wait()` joins them back).

    Receive buffers are allocated once per map slot and reused across steps; the
    full maps are views of them (rows [0, lines) of the concatenated strips)."""

    def __init__(self, plan: StripPlan, dist, dst: int = 0):
        self.plan, self.dist, self.dst = plan, dist, dst
        self.recv: dict[int, torch.Tensor] = {}
        self.works = []

    def padded(self, dtype, device) -> torch.Tensor:
        """A (per, samples) send buffer; the strip's rows are its first r1 - r0 rows."""
        return torch.zeros((self.plan.per, self.plan.samples), dtype=dtype, device=device)

    def launch(self, slot: int, send: torch.Tensor) -> None:
        p = self.plan
        if p.world == 1:
            return
        bufs = None
        if p.rank == self.dst:
            if slot not in self.recv:
                self.recv[slot] = torch.empty((p.world * p.per, p.samples), dtype=send.dtype,
                                              device=send.device)
            bufs = list(self.recv[slot].split(p.per))
        self.works.append(self.dist.gather(send, bufs, dst=self.dst, async_op=True))

    def wait(self) -> None:
        for w in self.works:
            w.wait()
        self.works.clear()

    def full(self, slot: int) -> torch.Tensor | None:
        if self.plan.rank != self.dst or slot not in self.recv:
            return None
        return self.recv[slot][: self.plan.lines]


def gather_maps(maps: Sequence[torch.Tensor], plan: StripPlan, dist, dst: int = 0):
    """Gather each rank's [r1-r0, samples] map to rank `dst` (padded to plan.per rows).
    Returns the full [lines, samples] maps on dst, None elsewhere."""
    g = MapGather(plan, dist, dst)
    for i, m in enumerate(maps):
        send = g.padded(m.dtype, m.device)
        send[: m.shape[0]].copy_(m)
        g.launch(i, send)
    g.wait()
    return [g.full(i) if plan.world > 1 else maps[i] for i in range(len(maps))]


def run_sharded(rows_of: Callable[[int, int], torch.Tensor], lines: int, samples: int,
                requests: Sequence[DetectRequest], dist, *,
                compute: Callable | None = None, order: int = 2, target_bands: int = 4):
    """Whole-image pipeline over `dist`'s ranks. rows_of(b0, b1) returns the full-band
    rows [b0, b1) (the host copy / generator) on this rank's device."""
    world, rank = dist.get_world_size(), dist.get_rank()
    plan = plan_strip(lines, samples, world, rank, requests)
    buf = rows_of(plan.b0, plan.b0 + plan.nb)
    compute = compute or compute_strip_gpu
    outs = compute(buf, plan, requests, order, target_bands)
    maps = gather_maps([s for s, _ in outs], plan, dist)
    counts = [c for _, c in outs]
    if any(c is not None for c in counts):
        cmaps = gather_maps([c if c is not None else torch.zeros((plan.r1 - plan.r0, samples),
                                                                 dtype=torch.int8, device=buf.device)
                             for c in counts], plan, dist)
    else:
        cmaps = [None] * len(requests)
    return plan, maps, cmaps


def pipeline_sharded(h_cube: torch.Tensor, order: int, target_bands: int,
                     requests: Sequence[DetectRequest], outputs, n_strips: int):
    """hsad_pipeline_sharded: one process, n_strips row strips dealt in contiguous blocks
    to the visible GPUs, host fp32 BIP cube in, host maps out (each GPU streams its own
    rows like hsad_pipeline_host; no collective). `outputs`: (scores, eigcount-or-None)
    CPU tensors."""
    import ctypes as C
    from . import _abi
    from .hsad import _check, _make_request
    if h_cube.is_cuda or h_cube.dtype != torch.float32:
        raise TypeError("h_cube must be a host float32 tensor")
    h_cube = h_cube.contiguous()
    lines, samples, bands = h_cube.shape
    reqs = (_abi.Request * len(requests))(*[_make_request(r, sc, cnt)
                                            for r, (sc, cnt) in zip(requests, outputs)])
    err = _abi.PixelError()
    _check(_abi.lib().hsad_pipeline_sharded(h_cube.data_ptr(), lines, samples, bands, order,
                                            target_bands, reqs, len(requests), n_strips,
                                            C.byref(err)), err)
    return outputs
