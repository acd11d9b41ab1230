"""hsad_gather_maps (NCCL score-map gather) and the streamed hsad_pipeline_sharded on one GPU.

Only one GPU is available to the tests: the gather runs at world size 1 over a real NCCL
communicator (hsad_nccl_comm_init_all), which exercises the run-time NCCL binding, the
strip plan and the root's in-place copy; the multi-rank send/recv offsets come from the
same hsad_strip_plan the gloo tests cover (tests/test_sharding_gloo.py)."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_1201_2025_b200")
from paper_1201_2025_b200 import _abi  # noqa: E402


def test_nccl_gather_world1_roundtrip():
    lib = _abi.lib()
    assert lib.hsad_nccl_available() == 0, lib.hsad_last_error_message()
    comm = C.c_void_p()
    assert lib.hsad_nccl_comm_init_all(C.byref(comm), 1) == 0, lib.hsad_last_error_message()
    try:
        lines, samples = 300, 129
        strip64 = torch.randn((lines, samples), dtype=torch.float64, device="cuda")
        strip8 = torch.randint(0, 4, (lines, samples), dtype=torch.int8, device="cuda")
        full64 = torch.zeros_like(strip64)
        full8 = torch.zeros_like(strip8)
        maps = (_abi.MapDesc * 2)(_abi.MapDesc(strip64.data_ptr(), full64.data_ptr(), 8),
                                  _abi.MapDesc(strip8.data_ptr(), full8.data_ptr(), 1))
        st = lib.hsad_gather_maps(comm, 1, 0, 0, lines, samples, maps, 2,
                                  torch.cuda.current_stream().cuda_stream)
        assert st == 0, lib.hsad_last_error_message()
        torch.cuda.synchronize()
        assert torch.equal(full64, strip64) and torch.equal(full8, strip8)
        # argument errors
        assert lib.hsad_gather_maps(comm, 2, 2, 0, lines, samples, maps, 2, None) == _abi.HSAD_E_INVALID_VALUE
        bad = (_abi.MapDesc * 1)(_abi.MapDesc(strip64.data_ptr(), None, 8))
        assert lib.hsad_gather_maps(comm, 1, 0, 0, lines, samples, bad, 1, None) == _abi.HSAD_E_INVALID_VALUE
    finally:
        assert lib.hsad_nccl_comm_destroy(comm) == 0


def test_nccl_map_gather_class_world1(orc):
    from paper_1201_2025_b200.sharded import NcclMapGather, plan_strip
    reqs = [hs.DetectRequest("lrx", hs.WindowConfig.single(7))]
    plan = plan_strip(64, 80, 1, 0, reqs)
    g = NcclMapGather(plan, dist=None)
    m = torch.rand((64, 80), dtype=torch.float64, device="cuda")
    g.launch(0, m)
    g.wait()
    torch.cuda.synchronize()
    assert torch.equal(g.full(0), m)
    g.close()
