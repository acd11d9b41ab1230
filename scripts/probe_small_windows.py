"""Small / sample-starved 4-band windows on uniform random cubes (test_window_sizes_and_borders
shapes): per case, pixels where the kernel and the fp64 oracle differ by > 1e-9, and how far
each is from the long-double value (oracle/hp_oracle.cpp)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1201_2025_b200 as hs  # noqa: E402

W1, W2 = hs.WindowConfig.single, hs.WindowConfig.dual
rows_out = []
for window, inner, outer in [(3, 1, 3), (7, 3, 9), (11, 5, 11), (15, 5, 15), (21, 7, 21), (25, 3, 25)]:
    for shape in ((23, 31), (6, 9), (40, 5)):
        cube = oracle.port.random_cube(*shape, 4, window * 7 + shape[0])
        g = torch.as_tensor(cube).cuda()
        (l, _), (d, _) = hs.detect_multi(g, [hs.DetectRequest("lrx", W1(window)),
                                             hs.DetectRequest("dwrx", W2(inner, outer))])
        l, d = l.cpu().numpy(), d.cpu().numpy()
        for name, got, want, hp in (
                (f"lrx {window}", l, oracle.port.local_rx(cube, window),
                 lambda r, c: oracle.port.hp_local_rx(cube, window, r, c)),
                (f"dwrx {inner}/{outer}", d, oracle.port.dwrx(cube, inner, outer),
                 lambda r, c: oracle.port.hp_dwrx(cube, inner, outer, r, c))):
            e = oracle.rel_diff(got, want)
            r, c = np.divmod(np.arange(got.size), got.shape[1])
            t, piv = hp(r, c)
            t = t.reshape(got.shape)
            eg, eo = oracle.rel_diff(got, t), oracle.rel_diff(want, t)
            rows_out.append({"case": name, "shape": shape, "max_gpu_vs_oracle": float(e.max()),
                             "max_gpu_vs_longdouble": float(eg.max()),
                             "max_oracle_vs_longdouble": float(eo.max()),
                             "px_gpu_vs_oracle_over_1e-9": int((e > 1e-9).sum()),
                             "px_gpu_vs_longdouble_over_1e-9": int((eg > 1e-9).sum()),
                             "max_pivot_ratio": float(piv.max())})
            print(json.dumps(rows_out[-1]), flush=True)
Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/small_windows.json").write_text(
    json.dumps(rows_out, indent=1))
