"""A/B probe over library builds: C5 sweep detector times per libhsad variant.

    python scripts/probe_libs.py variants/base.so variants/x.so ...   (each run twice, interleaved)
    an argument may carry environment settings: lib.so,HSAD_DWEST_SPLIT=1
Child mode (internal): HSAD_B200_LIB=<lib> python scripts/probe_libs.py --child
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SWEEP = [(3, 7), (5, 11), (5, 15), (7, 21)]


def child():
    sys.path.insert(0, str(ROOT))
    import torch
    import paper_1201_2025_b200 as hs
    from harness.scene import CONFIGS, generate_rows
    cfg = CONFIGS["C5"]
    cube = generate_rows(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], 0, cfg["lines"],
                         cfg["rate"], device="cuda")
    red = hs.reduce_cube(cube, 2, 4)
    del cube
    torch.cuda.empty_cache()
    W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
    line, tot, sums = [], 0.0, []
    for inner, outer in SWEEP:
        reqs = [hs.DetectRequest("lrx", W1(outer)), hs.DetectRequest("dwrx", W2(inner, outer)),
                hs.DetectRequest("dwest", W2(inner, outer), eigcount=True)]
        st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        outs = hs.detect_multi(red, reqs, status=st)
        for _ in range(3):
            hs.detect_multi(red, reqs, status=st, outputs=outs)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        ts = []
        for _ in range(10):
            s.record()
            hs.detect_multi(red, reqs, status=st, outputs=outs)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        td = ts[len(ts) // 2]
        tot += td
        line.append(f"{inner}/{outer} {td:.3f}")
        # checksum of the maps so variants can be compared for bit-identity
        sums.append(sum(float(o[0].double().sum()) for o in outs))
        sums.append(float(outs[2][1].double().sum()))
        # bit-level checksum (any differing bit changes it)
        sums.append(float(sum(int(o[0].contiguous().view(torch.int64).sum()) & 0xFFFFFFFFFFFF for o in outs)))
    print(f"{os.environ.get('PROBE_LABEL', Path(os.environ['HSAD_B200_LIB']).name):28s} " + "  ".join(line) + f"  sum {tot:.3f}",
          flush=True)
    print(f"{'':28s} checksums " + " ".join(f"{x:.15e}" for x in sums), flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["--child"]:
        child()
    else:
        for rep in range(2):
            for arg in sys.argv[1:]:
                lib, *kv = arg.split(",")
                env = dict(os.environ, HSAD_B200_LIB=str(Path(lib).resolve()), PROBE_LABEL=arg[-28:])
                env.update(x.split("=", 1) for x in kv)
                subprocess.run([sys.executable, __file__, "--child"], env=env, check=False)
