"""Summarise an ncu --set full report of one bench.py step (reduce + 4 detector launches)
into profiles/ncu_full_<tag>.json (selected metrics) and profiles/ncu_traffic_<tag>.json
(per-launch DRAM bytes, read by bench.py as roofline.traffic).

    python scripts/ncu_summary.py gpurun_out/prof_sweep_b.ncu-rep <tag> "<source note>"
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
LABELS = ["reduce (K1)", "detect 3/7", "detect 5/11", "detect 5/15", "detect 7/21"]
WINDOWS = ["3/7", "5/11", "5/15", "7/21"]


def label(i, name, seen):
    """reduce, then the detector launches in order; a '..., 1, 1>' detect kernel is the
    zero-window counting pass that follows each fast pass."""
    if "reduce" in name:
        return "reduce (K1)"
    if "detect_kernel_flagged<" in name:  # the counting pass over the tiles the fast pass flagged
        return f"detect {WINDOWS[(seen['fast'] - 1) % 4]} counting pass"
    args = name.split("detect_kernel<", 1)[1].split(">", 1)[0].replace("(bool)", "").replace("(int)", "")
    args = [a.strip() for a in args.split(",")]
    if len(args) >= 5 and args[4] in ("1", "true"):  # ZC: the zero-window counting pass
        return f"detect {WINDOWS[(seen['fast'] - 1) % 4]} counting pass"
    seen["fast"] += 1
    return f"detect {WINDOWS[(seen['fast'] - 1) % 4]}"


def main():
    rep, tag, note = sys.argv[1], sys.argv[2], sys.argv[3]
    first = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # window index of the first detect launch
    if rep.endswith(".csv"):  # already exported with ncu -i <rep> --page raw --csv
        raw = Path(rep).read_text()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    full, traffic = [], []
    seen = {"fast": first}
    for i, r in enumerate(rows[2:]):
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        if "hsad_b200" not in d["Kernel Name"]:  # torch fills of the probe script
            continue
        ent = {"kernel": d["Kernel Name"], "launch": label(i, d["Kernel Name"], seen)}
        for m in METRICS:
            ent[m] = d.get(m)
            ent[m + "_unit"] = u.get(m)
        full.append(ent)
        rb = float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
        wb = float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
        ms = float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "us" else 1.0)
        traffic.append({"launch": ent["launch"], "kernel": d["Kernel Name"][:60], "dram_read_bytes": rb,
                        "dram_write_bytes": wb, "ms": ms})
    src = f"profiles/ncu_full_{tag}.json ({note})"
    (ROOT / "profiles" / f"ncu_full_{tag}.json").write_text(
        json.dumps({"source": note, "c5_sweep_step": full}, indent=1))
    (ROOT / "profiles" / f"ncu_traffic_{tag}.json").write_text(
        json.dumps({"source": src, "launches": traffic}, indent=1))
    for t in traffic:
        print(f"{t['launch']:14s} {t['ms']:7.3f} ms  read {t['dram_read_bytes']/1e9:7.3f} GB  "
              f"write {t['dram_write_bytes']/1e9:6.3f} GB")


if __name__ == "__main__":
    main()
