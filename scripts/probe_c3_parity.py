"""C3 (100x100x189, no DWT) at the plain 1e-9 bar, every pixel, with a third opinion.

    python scripts/probe_c3_parity.py [out.json]

GPU maps (LRX 15 = the reference, the 15/5 guard extension, DWRX 5/15) against the fp64
oracle (oracle/hsad_oracle.cpp, explicit inverse like stats.cpp:31-62) and the
long-double restatement (oracle/hp_oracle.cpp) on all 10^4 pixels; per map: max rel_diff
of each pair, pixels over 1e-9, the LDL^T pivot-ratio (conditioning) distribution, and
the worst pixels with their 2-norm condition numbers (numpy).
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1201_2025_b200 as hs  # noqa: E402
from harness.scene import CONFIGS, generate_scene  # noqa: E402


def rel(a, b):
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def mirror(i, n):
    p = 2 * (n - 1)
    i = abs(i) % p
    return i if i < n else p - i


def cond2(cube, r, c, size, excl, ridge, inner=None):
    L, S, B = cube.shape
    h = size // 2
    xs = []
    for dr in range(-h, h + 1):
        for dc in range(-h, h + 1):
            if inner is not None:
                if abs(dr) <= inner // 2 and abs(dc) <= inner // 2:
                    continue
            elif abs(dr) <= excl // 2 and abs(dc) <= excl // 2:
                continue
            xs.append(cube[mirror(r + dr, L), mirror(c + dc, S)])
    X = np.array(xs, np.float64)
    C = np.cov(X.T, bias=True)
    C += ridge * np.trace(C) / B * np.eye(B)
    return float(np.linalg.cond(C))


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c3_parity.json"
    cfg = CONFIGS["C3"]
    cube, _ = generate_scene(cfg["lines"], cfg["samples"], cfg["bands"], cfg["seed"], cfg["rate"],
                             device="cuda")
    W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
    maps = hs.detect_multi(cube, [hs.DetectRequest("lrx", W1(15)),
                                  hs.DetectRequest("lrx", W1(15), guard=5),
                                  hs.DetectRequest("dwrx", W2(5, 15))])
    torch.cuda.synchronize()
    ch = cube.cpu().numpy()
    cores = os.cpu_count() or 1
    rows, cols = np.divmod(np.arange(100 * 100), 100)
    specs = [("lrx 15 (reference, guard 1)", lambda: oracle.port.local_rx(ch, 15, 1e-6, workers=cores),
              lambda: oracle.port.hp_local_rx(ch, 15, rows, cols, workers=cores), (15, 1, None)),
             ("lrx 15 guard 5 (extension)", lambda: oracle.port.local_rx(ch, 15, 1e-6, guard=5, workers=cores),
              lambda: oracle.port.hp_local_rx(ch, 15, rows, cols, guard=5, workers=cores), (15, 5, None)),
             ("dwrx 5/15", lambda: oracle.port.dwrx(ch, 5, 15, 1e-6, workers=cores),
              lambda: oracle.port.hp_dwrx(ch, 5, 15, rows, cols, workers=cores), (15, 0, 5))]
    res = {"config": "C3 100x100x189 fp32 BIP, no DWT, ridge 1e-6", "bar": 1e-9,
           "third_opinion": "oracle/hp_oracle.cpp: same algorithm in long double (eps 5.4e-20)",
           "maps": {}}
    for (name, fp64, hp, geo), (s, _) in zip(specs, maps):
        g = s.cpu().numpy()
        t0 = time.time()
        o = fp64()
        h, piv = hp()
        h = h.reshape(100, 100); piv = piv.reshape(100, 100)
        e_go, e_gh, e_oh = rel(g, o), rel(g, h), rel(o, h)
        worst = np.argsort(-e_go.ravel())[:12]
        res["maps"][name] = {
            "max_rel_gpu_vs_oracle": float(e_go.max()),
            "max_rel_gpu_vs_longdouble": float(e_gh.max()),
            "max_rel_oracle_vs_longdouble": float(e_oh.max()),
            "px_over_1e-9_gpu_vs_oracle": int((e_go > 1e-9).sum()),
            "px_over_1e-9_gpu_vs_longdouble": int((e_gh > 1e-9).sum()),
            "px_over_1e-9_oracle_vs_longdouble": int((e_oh > 1e-9).sum()),
            "px_where_oracle_is_closer_to_longdouble_than_gpu": int(((e_go > 1e-9) & (e_oh < e_gh)).sum()),
            "median_rel_gpu_vs_longdouble": float(np.median(e_gh)),
            "pivot_ratio_percentiles_50_90_99_max": [float(np.percentile(piv, q)) for q in (50, 90, 99, 100)],
            "worst_px_gpu_vs_oracle": [
                {"row": int(i // 100), "col": int(i % 100), "gpu_vs_oracle": float(e_go.ravel()[i]),
                 "gpu_vs_longdouble": float(e_gh.ravel()[i]), "oracle_vs_longdouble": float(e_oh.ravel()[i]),
                 "cond2": cond2(ch.astype(np.float64), int(i // 100), int(i % 100), geo[0], geo[1], 1e-6, geo[2])}
                for i in worst],
            "seconds_cpu": time.time() - t0}
        print(name, json.dumps({k: v for k, v in res["maps"][name].items() if k != "worst_px_gpu_vs_oracle"}),
              flush=True)
    Path(out_path).parent.mkdir(parents=True, exist_ok=True)
    Path(out_path).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
