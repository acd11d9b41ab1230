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
    q = row_quantum(lines, samples)
    per = -(-lines // (world * q)) * q
    r0, r1 = min(lines, rank * per), min(lines, (rank + 1) * per)
    b0, nb = strip_rows(lines, r0, r1, requests) if r1 > r0 else (r0, 0)
    return StripPlan(lines, samples, world, rank, q, per, r0, r1, b0, nb)


def compute_strip_gpu(buf: torch.Tensor, plan: StripPlan, requests: Sequence[DetectRequest],
                      order: int = 2, target_bands: int = 4, status: torch.Tensor | None = None):
    """DWT of the strip's buffer rows, then the fused detectors on rows [r0, r1)."""
    if plan.r1 <= plan.r0:
        return [(torch.empty((0, plan.samples), dtype=r.score_dtype, device=buf.device), None)
                for r in requests]
    red = reduce_cube(buf, order, target_bands) if order > 0 else buf
    return detect_multi(red, requests, lines=plan.lines, buf_row0=plan.b0,
                        row_begin=plan.r0, row_end=plan.r1, status=status)


def gather_maps(maps: Sequence[torch.Tensor], plan: StripPlan, dist, dst: int = 0):
    """Gather each rank's [r1-r0, samples] map to rank `dst` (padded to plan.per rows).
    Returns the full [lines, samples] maps on dst, None elsewhere."""
    out = []
    for m in maps:
        send = torch.zeros((plan.per, plan.samples), dtype=m.dtype, device=m.device)
        send[: m.shape[0]].copy_(m)
        bufs = ([torch.empty_like(send) for _ in range(plan.world)]
                if plan.rank == dst else None)
        dist.gather(send, bufs, dst=dst)
        out.append(torch.cat(bufs)[: plan.lines] if plan.rank == dst else None)
    return out


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
