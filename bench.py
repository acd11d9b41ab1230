"""Benchmark: Mpixel/s for DWT + LRX/DWRX/DWEST scoring (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

Workload (default C5, BASELINE.json configs[4]: the largest single-GPU config and the
one the 1/2/4/8-GPU scaling and HBM roofline are quoted on): a 4096 x 4096 x 224 fp32
BIP cube from the BASELINE generator (harness/scene.py, seeded, synthetic stand-in for
AVIRIS), db4 DWT to 4 approximation bands, then Local RX (11x11), DWRX (5/11) and
DWEST (5/11, + int8 eigen-count) — the fp64 path (all arithmetic fp64, fp64 score maps).

One step = one pass of that hot path over the cube:
  value : cube already resident in HBM; CUDA events around K steps of
          hsad_reduce + hsad_detect_multi (C-ABI) on the launching stream,
          barrier + synchronize on both sides, max over ranks;
  e2e   : hsad_pipeline_host (C-ABI) from pinned HOST memory: H2D of the cube,
          reduce, detectors, D2H of every map, timed per step (row strips on
          three streams, so the kernels and the D2H overlap the PCIe H2D).
Multi-GPU (torchrun): row strips aligned to hsad_row_quantum, each rank holds its
strip + mirror halo (generated from the same seeded row chunks = the host copy),
computes it, and the maps are gathered to rank 0 with NCCL through the product's C-ABI
(hsad_gather_maps: grouped ncclSend / ncclRecv straight into rank 0's full maps, one per
map, on a gather stream, so a window-pair group's maps travel while the next group's
detectors run; sharded.NcclMapGather) inside the timed region. scaling = "strong" (the 4096^2 image is fixed).

--impl reference times the CPU restatement of the reference (oracle/, the
reference itself needs Eigen3, absent here) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

PEAKS = ROOT / "MEASURED_PEAKS.json"
# BASELINE C5: DWT + all three detectors over the outer-window sweep 7, 11, 15, 21
# (inner 3 -> 7); LRX uses the outer window (guard 1, the reference's centre-only
# exclusion). (inner, outer) pairs:
SWEEP = [(3, 7), (5, 11), (5, 15), (7, 21)]
RMAX = max(o for _, o in SWEEP) // 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def hbm_peak():
    try:
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def requests(hs, score_dtype=torch.float64):
    W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
    reqs = []
    for inner, outer in SWEEP:
        reqs += [hs.DetectRequest("lrx", W1(outer), score_dtype=score_dtype),
                 hs.DetectRequest("dwrx", W2(inner, outer), score_dtype=score_dtype),
                 hs.DetectRequest("dwest", W2(inner, outer), eigcount=True, score_dtype=score_dtype)]
    return reqs


def bytes_per_pixel(bands: int) -> int:
    # algorithmic: read the fp32 spectrum once, write 12 fp64 maps + 4 int8 eigen-counts
    return 4 * bands + len(SWEEP) * (3 * 8 + 1)


def oracle_step(oracle, cube_np, n, cores):
    """DWT of the rows the windows of output rows [0, n) need + the 12 detector maps."""
    red = oracle.port.reduce_cube(cube_np[: min(cube_np.shape[0], n + 2 * RMAX + 1)], 2, 4,
                                  workers=cores)
    for inner, outer in SWEEP:
        oracle.port.local_rx(red, outer, 1e-6, workers=cores, rows=(0, n))
        oracle.port.dwrx(red, inner, outer, 1e-6, workers=cores, rows=(0, n))
        oracle.port.dwest(red, inner, outer, 0.1, workers=cores, rows=(0, n))


def cpu_baseline(cube_rows_np: np.ndarray, lines: int, rows_total: int, budget_s: float):
    """Oracle port (the CPU restatement of proj/core/src/{wavelet,detect,stats}.cpp)
    on a bounded row sample of the same cube, all host threads."""
    import oracle
    cores = os.cpu_count() or 1
    L = cube_rows_np.shape[0]
    # the sample: rows [0, n) of the workload, DWT of the rows the windows need
    def run(n):
        t0 = time.perf_counter()
        oracle_step(oracle, cube_rows_np, n, cores)
        return time.perf_counter() - t0
    n, dt = 8, 0.0
    for _ in range(3):  # grow the sample until it takes ~budget_s (or uses every row)
        dt = run(n)
        if dt >= 0.6 * budget_s or n >= L - 2 * RMAX - 1:
            break
        n = int(max(8, min(L - 2 * RMAX - 1, n * budget_s / max(dt, 1e-3))))
    px = n * cube_rows_np.shape[1]
    return {"value": px / dt / 1e6, "unit": "Mpixel/s", "cores": cores, "kind": "port",
            "sample": f"rows 0..{n} of the workload ({px} px; DWT on {min(L, n + 2 * RMAX + 1)} rows "
                      f"+ LRX/DWRX/DWEST at 4 window pairs), {dt:.1f} s, oracle/hsad_oracle.cpp "
                      f"with {cores} threads"}


# ---- parity gate on the benchmarked workload (a deterministic subset) ----------

def mirror(i: int, n: int) -> int:
    """mirror_index (proj/core/src/detect.cpp:71-76)."""
    if n == 1:
        return 0
    p = 2 * (n - 1)
    i = abs(i) % p
    return i if i < n else p - i


def parity_rows(lines: int, quantum: int, rmax: int = RMAX, n_random: int = 64,
                seed: int = 0x1201) -> list[int]:
    """SURVEY 8d's C5 subset: the top border rows 0..R+q (the first chunk and its
    warm-up), every shard-boundary row +-R for G in {2, 4, 8}, the last row of a few
    chunks (longest running-sum chain), n_random seeded random rows, the last R+1 rows."""
    rows = set(range(0, min(lines, rmax + quantum + 1)))
    for g in (2, 4, 8):
        per = -(-lines // (g * quantum)) * quantum
        for k in range(1, g):
            b = k * per
            rows.update(r for r in range(b - rmax, b + rmax + 1) if 0 <= r < lines)
    rows.update(r for r in (quantum - 1, 2 * quantum - 1, lines // 2 - 1) if 0 <= r < lines)
    rng = np.random.default_rng(seed)
    rows.update(int(r) for r in rng.integers(0, lines, n_random))
    rows.update(range(max(0, lines - rmax - 1), lines))
    return sorted(rows)


def runs_of(rows):
    out, s = [], None
    for i, r in enumerate(rows):
        if s is None:
            s = r
        if i + 1 == len(rows) or rows[i + 1] != r + 1:
            out.append((s, r + 1))
            s = None
    return out


def topk_check(gpu: np.ndarray, ref: np.ndarray, k: int):
    """Identical top-k pixel sets (k = truth positives), plus the oracle's k/k+1 margin."""
    if k <= 0 or k >= gpu.size:
        return True, None
    g = np.argsort(-gpu.ravel(), kind="stable")[:k]
    o_order = np.argsort(-ref.ravel(), kind="stable")
    o = o_order[:k]
    margin = float(ref.ravel()[o_order[k - 1]] - ref.ravel()[o_order[k]])
    return bool(set(g.tolist()) == set(o.tolist())), margin


def oracle_parity(host_cube: np.ndarray, lines: int, rows: list[int], reduced_gpu_rows,
                  maps_gpu_rows, truth_rows: np.ndarray, cores: int, rmax: int = RMAX,
                  sweep=SWEEP):
    """Compares the GPU step's outputs on `rows` with the oracle (oracle/hsad_oracle.cpp).

    host_cube: the fp32 (lines, samples, bands) input; reduced_gpu_rows(r0, r1) -> the
    GPU's reduced rows; maps_gpu_rows[i](rows) -> map i on `rows` ((scores, counts|None)
    in the order of requests()). Returns the JSON `parity` block."""
    import oracle
    t0 = time.perf_counter()
    samples = host_cube.shape[1]
    need = sorted({mirror(r + d, lines) for r in rows for d in range(-rmax, rmax + 1)})
    red = np.zeros((lines, samples, 4), np.float64)
    dwt_err = 0.0
    for a, b in runs_of(need):
        red[a:b] = oracle.port.reduce_cube(host_cube[a:b], 2, 4, workers=cores)
        dwt_err = max(dwt_err, oracle.max_rel_diff(reduced_gpu_rows(a, b), red[a:b]))
    runs = runs_of(rows)
    names, errs, cnt_bad, topk, ties = [], [], [], [], {}
    i = 0
    for inner, outer in sweep:
        ref_maps = [np.concatenate([oracle.port.local_rx(red, outer, 1e-6, workers=cores, rows=ab)
                                    for ab in runs]),
                    np.concatenate([oracle.port.dwrx(red, inner, outer, 1e-6, workers=cores, rows=ab)
                                    for ab in runs])]
        ds = [oracle.port.dwest(red, inner, outer, 0.1, workers=cores, rows=ab) for ab in runs]
        ref_maps.append(np.concatenate([s for s, _ in ds]))
        ref_cnt = np.concatenate([c for _, c in ds])
        for algo, ref in zip(("lrx", "dwrx", "dwest"), ref_maps):
            gs, gc = maps_gpu_rows[i](rows)
            names.append(f"{algo} {inner}/{outer}" if algo != "lrx" else f"lrx {outer}")
            errs.append(oracle.max_rel_diff(gs, ref))
            same, margin = topk_check(gs, ref, int(truth_rows.sum()))
            topk.append({"identical": same, "oracle_k_margin": margin})
            if gc is not None:
                cnt_bad.append(int((gc != ref_cnt).sum()))
            i += 1
        mg = [oracle.port.dwest_margins(red, inner, outer, 0.1, workers=cores, rows=ab)
              for ab in runs]
        cm = np.concatenate([c for c, _ in mg])
        sm = np.concatenate([s for _, s in mg])
        ties[f"{inner}/{outer}"] = {"cutoff_margin_lt_1e-12": int((cm < 1e-12).sum()),
                                    "sign_margin_lt_1e-12": int((sm < 1e-12).sum()),
                                    "cutoff_margin_lt_1e-9": int((cm < 1e-9).sum()),
                                    "min_cutoff_margin": float(cm.min()),
                                    "min_sign_margin": float(sm.min())}
    npx = len(rows) * samples
    gate = (dwt_err <= 1e-5 and max(errs) <= 1e-9 and not any(cnt_bad)
            and all(t["identical"] for t in topk))
    return {"pass": bool(gate), "rows": len(rows), "pixels": npx,
            "row_set": "0..R+q, shard boundaries +-R for G in {2,4,8}, chunk ends, "
                       "64 seeded random rows, last R+1 rows (SURVEY 8d)",
            "dwt_max_rel_diff": dwt_err,
            "max_rel_diff": dict(zip(names, errs)),
            "bar": "rel_diff |a-b|/max(1,|a|,|b|) (testutil.hpp:34-36) <= 1e-9 fp64 maps, "
                   "DWT <= 1e-5, identical eigen-counts and top-k",
            "eigcount_mismatches": cnt_bad,
            "topk_identical": [t["identical"] for t in topk],
            "topk_k": int(truth_rows.sum()),
            "topk_oracle_margin_min": min((t["oracle_k_margin"] for t in topk
                                           if t["oracle_k_margin"] is not None), default=None),
            "dwest_near_ties": ties,
            "oracle": "oracle/hsad_oracle.cpp (pinned to the reference's own code, tests/test_oracle_pin.py)",
            "seconds": time.perf_counter() - t0}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU restatement of the reference path (the reference's
    Eigen build cannot be compiled here) on the host cores, on the same bytes as the
    GPU arm (host generator) and the same workload. A step is a bounded sample: the
    DWT of the rows the sample's windows need (timed, then scaled to the sample's own
    rows so halo rows are not over-counted) + the 12 maps of 8 border and 8 interior
    output rows."""
    if rank != 0:
        return
    from harness.scene import generate_rows_np
    import oracle
    cores = os.cpu_count() or 1
    lines, samples, bands = cfg["lines"], cfg["samples"], cfg["bands"]
    half = 32
    mid = lines // 2
    bands_rows = [(0, half), (mid, mid + half)]  # border rows and interior rows
    cubes = []
    for a, b in bands_rows:
        lo, hi = max(0, a - RMAX), min(lines, b + RMAX)
        cubes.append((a - lo, b - lo, generate_rows_np(lines, samples, bands, cfg["seed"], lo, hi,
                                                      cfg["rate"])))
    n_out = sum(b - a for a, b in bands_rows)

    def step():
        t_red = t_det = 0.0
        for a, b, cube in cubes:
            t0 = time.perf_counter()
            red = oracle.port.reduce_cube(cube, 2, 4, workers=cores)
            t1 = time.perf_counter()
            for inner, outer in SWEEP:
                oracle.port.local_rx(red, outer, 1e-6, workers=cores, rows=(a, b))
                oracle.port.dwrx(red, inner, outer, 1e-6, workers=cores, rows=(a, b))
                oracle.port.dwest(red, inner, outer, 0.1, workers=cores, rows=(a, b))
            t2 = time.perf_counter()
            t_red += (t1 - t0) * (b - a) / cube.shape[0]  # DWT cost of the output rows only
            t_det += t2 - t1
        return t_red + t_det

    for _ in range(args.warmup):
        step()
    dt = sum(step() for _ in range(args.steps)) / args.steps
    px = n_out * samples
    v = px / dt / 1e6
    line = {
        "impl": "reference", "metric": "Mpixels/sec for DWT+LRX/DWRX/DWEST scoring",
        "value": v, "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": run_config(args, cfg, world),
        "cpu_baseline": {"value": v, "unit": "Mpixel/s", "cores": cores, "kind": "port",
                         "sample": f"per step: output rows {bands_rows} ({px} px, border + interior) "
                                   f"x 12 maps (LRX/DWRX/DWEST at 4 window pairs) + their DWT "
                                   f"(timed on the rows the windows need, scaled to the output "
                                   f"rows); same bytes as the GPU arm (harness/scene_gen.cpp); "
                                   f"CPU restatement oracle/hsad_oracle.cpp, {cores} threads "
                                   f"(the reference needs Eigen3, absent)"},
        "e2e": {"value": v, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def detector_ncu():
    """Issue-active and fp64-pipe utilisation of the four detector launches from the
    committed ncu --set full capture of this workload (the detectors' own roofline is
    fp64 issue, not HBM: ~57 B/px of DRAM traffic per launch)."""
    f = ROOT / "profiles" / "ncu_full_r2b_sweep.json"
    if not f.exists():
        return {}
    d = json.loads(f.read_text())
    order = ["detect 3/7", "detect 5/11", "detect 5/15", "detect 7/21"]
    det = sorted((k for k in d["c5_sweep_step"] if k["launch"] in order),
                 key=lambda k: order.index(k["launch"]))
    key_i = "smsp__issue_active.avg.pct_of_peak_sustained_active"
    key_f = "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
    def fp64_tflops(k):  # executed fp64 flops (2 per DFMA) per elapsed cycle x SM clock
        m = "smsp__sass_thread_inst_executed_op_{}_pred_on.sum.per_cycle_elapsed"
        try:
            f = 2 * float(k[m.format("dfma")]) + float(k[m.format("dadd")]) + float(k[m.format("dmul")])
        except (KeyError, TypeError, ValueError):
            return None
        return round(f * 1.965e9 / 1e12, 2)
    peak_file = ROOT / "profiles" / "fp64_peak_r2.json"
    try:
        fp64_peak = json.loads(peak_file.read_text())["dfma_tflops"]
        peak_src = f"{peak_file.relative_to(ROOT)} (harness/peaks/fp64_peak.cu on a B200)"
    except Exception:
        fp64_peak, peak_src = None, "profiles/fp64_peak_r2.json missing"
    return {"ncu_issue_active_frac": [round(float(k[key_i]) / 100, 3) for k in det],
            "ncu_fp64_pipe_frac": [round(float(k[key_f]) / 100, 3) for k in det],
            "ncu_fp64_tflops_executed": [fp64_tflops(k) for k in det],
            "fp64_peak_tflops_measured": fp64_peak, "fp64_peak_source": peak_src,
            "ncu_source": "profiles/ncu_full_r2b_sweep.json (fast passes of the 7/3, 11/5, 15/5, 21/7 detectors)"}


def run_config(args, cfg, world):
    """`config` of both arms (identical keys and values: the driver compares them)."""
    return dict(workload_config(args, cfg), parallelism=f"row-strips x{world}")


def workload_config(args, cfg):
    sweep = ", ".join(f"{i}/{o}" for i, o in SWEEP)
    return {"workload": f"{args.config}: {cfg['lines']}x{cfg['samples']}x{cfg['bands']} fp32 BIP, "
                        f"db4 DWT->4 bands + LRX/DWRX/DWEST (+DWEST eigen-count) at each "
                        f"inner/outer window of the sweep {sweep} (LRX on the outer window): "
                        f"12 fp64 maps per step",
            "window_sweep": [{"inner": i, "outer": o} for i, o in SWEEP],
            "lines": cfg["lines"], "samples": cfg["samples"], "bands": cfg["bands"],
            "seed": cfg["seed"], "anomaly_rate": cfg["rate"],
            "l2": "inputs larger than L2 (15 GB cube vs 126 MB L2)" if args.config == "C5"
                  else "see note: L2 flushed between steps"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from harness.scene import CONFIGS
    cfg = CONFIGS[args.config]
    dist = None
    if world > 1:
        # the communicator set-up lines ("... nranks N ...") show the rank count in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        if args.impl == "b200":  # the reference arm is CPU-only (gloo)
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "b200" else "gloo")
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        if dist is not None:
            dist.destroy_process_group()
        return
    run_b200(args, cfg, rank, world, local, dist)
    if dist is not None:
        dist.destroy_process_group()


def run_b200(args, cfg, rank, world, local, dist):
    import paper_1201_2025_b200 as hs
    from harness.scene import generate_rows
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    lines, samples, bands = cfg["lines"], cfg["samples"], cfg["bands"]
    reqs = requests(hs)

    # ---- row strip of this rank (aligned to the detector row quantum) + halo
    from paper_1201_2025_b200.sharded import plan_strip
    plan = plan_strip(lines, samples, world, rank, reqs)
    q, per, r0, r1, b0, nb = plan.quantum, plan.per, plan.r0, plan.r1, plan.b0, plan.nb
    # the strip's rows are generated on the host (identical bytes to the reference arm and
    # the parity oracle) into pinned memory: the e2e leg streams from this copy
    host_cube = generate_rows(lines, samples, bands, cfg["seed"], b0, b0 + nb, cfg["rate"],
                              pin=True)
    cube = host_cube.to(dev)
    red = torch.empty((nb, samples, 4), dtype=torch.float64, device=dev)
    # maps live in padded (per, samples) buffers: the strip's rows come first, so at N > 1
    # they are the NCCL send buffers themselves (no staging copy)
    from paper_1201_2025_b200.sharded import MapGather, NcclMapGather
    # the product's C-ABI NCCL gather (hsad_gather_maps) on its own communicator;
    # HSAD_TORCH_GATHER=1 uses torch.distributed.gather instead
    gather = None
    if world > 1:
        if os.environ.get("HSAD_TORCH_GATHER"):
            gather = MapGather(plan, dist)
        else:
            # every rank must take the same route: agree on whether the library's communicator came up
            try:
                gather, ok = NcclMapGather(plan, dist), 1
            except Exception as e:  # e.g. no loadable libnccl.so.2 for the C-ABI on this box
                print(f"[bench] hsad_gather_maps unavailable on rank {rank} ({e}); using torch.distributed.gather",
                      file=sys.stderr, flush=True)
                gather, ok = None, 0
            flag = torch.tensor([ok], device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                gather = MapGather(plan, dist)
    pad = lambda dt: torch.zeros((max(per, r1 - r0), samples), dtype=dt, device=dev)  # noqa: E731
    outs_pad = [(pad(torch.float64), pad(torch.int8) if r.eigcount else None) for r in reqs]
    outs = [(sc[: r1 - r0], None if cnt is None else cnt[: r1 - r0]) for sc, cnt in outs_pad]
    status = torch.full((1,), -1, dtype=torch.int64, device=dev)

    lib = hs._abi.lib()
    import ctypes as C
    stream = torch.cuda.current_stream(dev)
    # one request group per window pair of the sweep (3 requests: one fused launch each),
    # so at N > 1 the maps of a finished group are gathered while the next group computes
    per_group = len(reqs) // len(SWEEP)
    groups = []
    for g in range(len(SWEEP)):
        sl = slice(g * per_group, (g + 1) * per_group)
        groups.append(((hs._abi.Request * per_group)(*[
            hs.hsad._make_request(r, sc, cnt) for r, (sc, cnt) in zip(reqs[sl], outs[sl])]),
            list(range(sl.start, sl.stop))))
    # N = 1: the whole sweep in one hsad_reduce_detect call (12 requests = 4 groups); the
    # library forks groups 1.. onto side streams right after the reduction, next to group 0
    # (widest window pair first: the longest launch starts first and the shorter ones fill its
    # tail; every request carries its own output pointers, so the order only affects timing)
    order = [i for g in reversed(range(len(SWEEP))) for i in range(g * per_group, (g + 1) * per_group)]
    all_creqs = (hs._abi.Request * len(reqs))(*[
        hs.hsad._make_request(reqs[i], outs[i][0], outs[i][1]) for i in order])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    kern_ms = {"first": [], "rest": []}
    fused = []

    def step(record=False):
        if gather is None and not record:
            st = lib.hsad_reduce_detect(cube.data_ptr(), lines, samples, bands, 2, 4, b0, nb, r0, r1,
                                        red.data_ptr(), all_creqs, len(reqs), status.data_ptr(), None,
                                        stream.cuda_stream)
            assert st == 0, lib.hsad_last_error_message()
            return
        # (per-kernel timing pass, and N > 1 where each group's maps are gathered as it ends)
        # the DWT and the first window pair's detectors in one call: the reduction folds
        # into that launch (hsad_reduce_detect; hsad_reduce runs first when it cannot,
        # e.g. a strip halo wider than the first windows)
        creqs, idx = groups[0]
        st = lib.hsad_reduce_detect(cube.data_ptr(), lines, samples, bands, 2, 4, b0, nb, r0, r1,
                                    red.data_ptr(), creqs, len(idx), status.data_ptr(), None,
                                    stream.cuda_stream)
        assert st == 0, lib.hsad_last_error_message()
        fused.append(lib.hsad_last_reduce_detect_fused())
        if record:
            ev[1].record(stream)
        for gi, (creqs, idx) in enumerate(groups):
            if gi > 0:
                st = lib.hsad_detect_multi(red.data_ptr(), 8, lines, samples, 4, b0, nb, r0, r1, creqs,
                                           len(idx), status.data_ptr(), None, stream.cuda_stream)
                assert st == 0, lib.hsad_last_error_message()
            if gather is not None:  # NCCL gather of this group's maps, overlapping the next group
                src = outs_pad if isinstance(gather, MapGather) else outs
                for i in idx:
                    gather.launch(2 * i, src[i][0])
                    if src[i][1] is not None:
                        gather.launch(2 * i + 1, src[i][1])
        if record:
            ev[2].record(stream)
        if gather is not None:
            gather.wait()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # per-kernel durations (events on the launching stream), outside the headline timing
    for _ in range(3):
        ev[0].record(stream)
        step(record=True)
        ev[2].synchronize()
        kern_ms["first"].append(ev[0].elapsed_time(ev[1]))
        kern_ms["rest"].append(ev[1].elapsed_time(ev[2]))

    clocks = Clocks(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        step()
    end.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    bad = int(status.item())
    assert bad == -1, f"per-pixel failure recorded: {bad}"

    # ---- end to end through the C-ABI from pinned host buffers (rank 0 strip only at N>1)
    e2e = None
    host_out = None
    if rank == 0 or world == 1:
        host_out = [(torch.empty((nb, samples), dtype=torch.float64, pin_memory=True),
                     torch.empty((nb, samples), dtype=torch.int8, pin_memory=True) if r.eigcount
                     else None) for r in reqs]
        hs.pipeline_host(host_cube, 2, 4, reqs, host_out)  # warm (allocates the device cache)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            hs.pipeline_host(host_cube, 2, 4, reqs, host_out)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        h2d = nb * samples * bands * 4
        # PCIe ceiling: one plain pinned H2D copy of the same cube
        dev_copy = torch.empty_like(host_cube, device=dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dev_copy.copy_(host_cube, non_blocking=True)
        torch.cuda.synchronize()
        h2d_only_s = time.perf_counter() - t1
        del dev_copy
        d2h = sum(nb * samples * (8 + (1 if r.eigcount else 0)) for r in reqs)
        e2e = {"value": nb * samples / e2e_s / 1e6, "unit": "Mpixel/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_s * 1e3,
               "h2d_only_ms": h2d_only_s * 1e3,
               "h2d_gbs": h2d / h2d_only_s / 1e9,
               "bound": "PCIe: the fp32 cube H2D; reduce, detectors and map D2H run under it "
                        "in row strips (hsad_pipeline_host)",
               "path": "hsad_pipeline_host (C-ABI): pinned host cube -> row-strip pipelined "
                       "H2D / reduce / fused detectors / D2H" +
                       (f" (rank 0 strip, {nb} rows)" if world > 1 else "")}

    if rank != 0:
        return
    total_px = lines * samples
    value = total_px / (ms_step / 1e3) / 1e6
    peak, peak_src = hbm_peak()
    bpp = bytes_per_pixel(bands)
    first_ms = statistics.median(kern_ms["first"])
    rest_ms = statistics.median(kern_ms["rest"])
    local_px = (r1 - r0) * samples
    is_fused = bool(fused[-1])
    first_gbs = nb * samples * (bands * 4 + 32 + 3 * 8 + 1) / (first_ms / 1e3) / 1e9
    step_gbs = value * 1e6 * bpp / 1e9
    # DRAM traffic per launch from the committed ncu --set full capture of this workload
    traffic, traffic_src = None, None
    tfile = ROOT / "profiles" / "ncu_traffic_r2b_sweep.json"
    if args.config == "C5" and world == 1 and tfile.exists():
        tj = json.loads(tfile.read_text())
        traffic = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in tj["launches"]) / 1e9
        traffic_src = f"GB per step (reduce + 4 detector fast passes + 4 counting passes), {tj['source']}"
    line = {
        "metric": "Mpixels/sec for DWT+LRX/DWRX/DWEST scoring",
        "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": run_config(args, cfg, world),
        "launch": {"row_quantum": q, "strip_rows": per,
                   "groups": ("one hsad_reduce_detect call, window-pair groups 1.. forked onto side "
                              "streams after the reduction" if gather is None else
                              "one call per window-pair group, maps gathered as each group ends")},
        "roofline": {
            "bound": "hbm", "achieved": step_gbs, "peak": peak, "unit": "GB/s",
            "frac": step_gbs / peak, "traffic": traffic, "traffic_unit": traffic_src,
            "algorithmic_gb_per_step": bpp * total_px / 1e9 / world,
            "basis": f"whole step, algorithmic {bpp} B/px (4L fp32 read + 12 fp64 maps + 4 int8 "
                     f"counts) x px/s, {peak_src}",
            "kernels": {
                ("DWT fused into the 3/7 detector launch (hsad_reduce_detect)" if is_fused else
                 "reduce (K1) + 3/7 detectors"): {
                    "ms": first_ms, "achieved_gbs": first_gbs, "frac": first_gbs / peak,
                    "share": first_ms / (first_ms + rest_ms), "fused": is_fused,
                    "bytes": "fp32 cube read + fp64 reduced write + 3 fp64 maps + 1 int8 map"},
                "detect 5/11, 5/15, 7/21 (K2-K4, 3 launches, fp64-compute-bound)": dict(
                    {"ms": rest_ms, "share": rest_ms / (first_ms + rest_ms),
                     "px_per_s": local_px / (rest_ms / 3 / 1e3)}, **detector_ncu()),
            },
        },
        "clocks": clk,
        # per step: per window pair a fast detector pass and its zero-window counting pass
        # (which exits at once on data without all-zero spectra and repairs ill-conditioned
        # pixels); K1 only when the reduction could not be fused into the first pass
        "gpu_launches": ((0 if is_fused else 1) + 2 * len(SWEEP)) * args.steps,
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(host_cube.numpy(), lines, nb, args.cpu_seconds)
    if world == 1 and not args.no_parity:
        from harness.scene import anomaly_fill
        rows = parity_rows(lines, q)
        idx = torch.tensor(rows)
        truth, _ = anomaly_fill(lines, samples, cfg["rate"], cfg["seed"])
        maps = []
        for (sc, cnt), (hsc, hcnt) in zip(outs, host_out):
            def get(rws, sc=sc, cnt=cnt):
                return (sc[idx.to(dev)].cpu().numpy(),
                        None if cnt is None else cnt[idx.to(dev)].cpu().numpy())
            maps.append(get)
        par = oracle_parity(host_cube.numpy(), lines, rows,
                            lambda a, b: red[a:b].cpu().numpy(), maps, truth[rows],
                            os.cpu_count() or 1)
        # the e2e leg (hsad_pipeline_host, pinned host buffers) must reproduce the
        # device-resident maps bit for bit (quantum-aligned row strips)
        par["e2e_maps_bit_identical"] = all(
            torch.equal(sc.cpu(), hsc) and (cnt is None or torch.equal(cnt.cpu(), hcnt))
            for (sc, cnt), (hsc, hcnt) in zip(outs, host_out))
        par["pass"] = par["pass"] and par["e2e_maps_bit_identical"]
        line["parity"] = par
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
