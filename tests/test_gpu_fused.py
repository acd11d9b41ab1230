"""Fused DWT -> detector launch (opt-in: HSAD_FUSE=1) against the two-step path.

hsad_reduce_detect folds the reduction into its first detector launch when the launch's
windows read exactly the buffer rows (fused_dwt_row: every CTA computes the reduced rows
of its strip, warm-up rows first, then each entering row one step ahead of the TMA copy
that reads it, with hsad_reduce's exact lane-split arithmetic). The reduced cube and every
map must be bit-identical to hsad_reduce followed by hsad_detect_multi, on images with
mirrored borders, several row chunks and column strips, and the C5 launch shape.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_1201_2025_b200")
from paper_1201_2025_b200 import _abi  # noqa: E402


@pytest.fixture(autouse=True)
def _fuse_on(monkeypatch):
    """The fused launch is opt-in (HSAD_FUSE=1; measured slower than two steps)."""
    monkeypatch.setenv("HSAD_FUSE", "1")

DEV = "cuda:0"


def W1(n):
    return hs.WindowConfig.single(n)


def W2(i, o):
    return hs.WindowConfig.dual(i, o)


def trio(inner, outer):
    return [hs.DetectRequest("lrx", W1(outer)), hs.DetectRequest("dwrx", W2(inner, outer)),
            hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)]


def check_fused(cube, reqs, expect_fused=True):
    red, outs = hs.reduce_detect(cube, reqs, 2, 4)
    torch.cuda.synchronize()
    fused = _abi.lib().hsad_last_reduce_detect_fused()
    assert fused == int(expect_fused)
    red2 = hs.reduce_cube(cube, 2, 4)
    two = hs.detect_multi(red2, reqs)
    torch.cuda.synchronize()
    assert torch.equal(red, red2)
    for (a, ac), (b, bc) in zip(outs, two):
        assert torch.equal(a, b)
        if ac is not None:
            assert torch.equal(ac, bc)


@pytest.mark.parametrize("lines,samples,bands", [(9, 11, 189), (70, 300, 224), (150, 129, 64),
                                                 (203, 520, 224), (40, 2100, 189)])
def test_fused_equals_two_step(orc, lines, samples, bands):
    cube = torch.as_tensor(orc.port.random_cube(lines, samples, bands, lines * 7 + samples)
                           .astype(np.float32)).to(DEV)
    check_fused(cube, trio(3, 7))


def test_fused_then_more_groups_equals_two_step(orc):
    """The C5 request list: the first window pair's launch carries the reduction, the
    other three groups read the reduced rows it wrote."""
    cube = torch.as_tensor(orc.port.random_cube(96, 333, 224, 91).astype(np.float32)).to(DEV)
    reqs = []
    for i, o in [(3, 7), (5, 11), (5, 15), (7, 21)]:
        reqs += trio(i, o)
    check_fused(cube, reqs)


def test_not_fused_when_buffer_is_wider_than_the_windows(orc):
    """A strip buffer with a halo wider than the first group's windows: the rows outside
    them are reduced by hsad_reduce first (same results)."""
    lines, samples = 120, 90
    full = torch.as_tensor(orc.port.random_cube(lines, samples, 64, 92).astype(np.float32)).to(DEV)
    reqs = trio(3, 7) + trio(5, 11)
    r0, r1 = 40, 80
    b0, nb = hs.strip_rows(lines, r0, r1, reqs)
    buf = full[b0:b0 + nb].contiguous()
    red, outs = hs.reduce_detect(buf, reqs, 2, 4, lines=lines, buf_row0=b0, row_begin=r0, row_end=r1)
    assert _abi.lib().hsad_last_reduce_detect_fused() == 0
    whole = hs.detect_multi(hs.reduce_cube(full, 2, 4), reqs)
    for (a, _), (b, _) in zip(outs, whole):
        assert torch.equal(a, b[r0:r1])


def test_fused_c5_launch_shape(orc):
    """C5 geometry (4096 columns, 224 bands, row quantum 32) on the smallest such image."""
    from harness.scene import CONFIGS, generate_rows
    cfg = CONFIGS["C5"]
    q5 = hs.row_quantum(4096, 4096)
    lines = q5
    while hs.row_quantum(lines, 4096) != q5:
        lines += q5
    cube = generate_rows(lines, 4096, 224, cfg["seed"], 0, lines, cfg["rate"], device=DEV)
    check_fused(cube, trio(3, 7) + trio(5, 11))
