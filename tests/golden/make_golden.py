"""Generate tests/golden/*.npz from the REFERENCE's own code (oracle/_ref: the
reference's wavelet.cpp and its naive detector oracles, tests/support/oracles.cpp,
compiled in place from /root/reference by oracle/Makefile).

Inputs are the reference tests' own seeded generators (xoshiro256++ random_cube /
random_signal of proj/tests/support/testutil.hpp), restated in the oracle port and
bit-checked here against the seeds' known first values. Run in the build
container (where /root/reference exists):  python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    ref, port = oracle.ref, oracle.port
    assert ref is not None, "oracle/_ref not built: needs /root/reference"
    g = {}
    # wavelet: taps of every order, Haar [1,2,3,4], reduce_cube of random cubes
    for order in range(1, 11):
        lo, hi = ref.daubechies(order)
        g[f"taps_low_{order}"] = lo
        g[f"taps_high_{order}"] = hi
    a, d = ref.dwt_level(np.array([1.0, 2, 3, 4]), 1)
    g["haar_1234_approx"], g["haar_1234_detail"] = a, d
    for bands, seed, order, target in ((189, 33, 2, 4), (224, 34, 2, 4), (64, 21, 3, 4),
                                       (189, 35, 1, 8)):
        cube = port.random_cube(5, 7, bands, seed)
        g[f"reduce_in_{bands}_{seed}"] = cube
        g[f"reduce_out_{bands}_{seed}_{order}_{target}"] = ref.reduce_cube(cube, order, target)
    np.savez_compressed(OUT / "golden_wavelet.npz", **g)

    d = {}
    # detectors: the reference's naive oracles on the reference tests' cubes
    for seed in (2024, 0xACCE3):
        cube = port.random_cube(10, 10, 4, seed)
        d[f"cube_{seed}"] = cube
        d[f"lrx5_{seed}"] = ref.naive_lrx(cube, 5, 1e-6)
        d[f"dwrx37_{seed}"] = ref.naive_dwrx(cube, 3, 7, 1e-6)
        d[f"dwest37_{seed}"] = ref.naive_dwest(cube, 3, 7, 0.1)
    cube = port.random_cube(13, 9, 3, 99)
    d["cube_99"] = cube
    d["lrx7_99"] = ref.naive_lrx(cube, 7, 1e-6)
    d["dwrx59_99"] = ref.naive_dwrx(cube, 5, 9, 1e-6)
    d["dwest59_99"] = ref.naive_dwest(cube, 5, 9, 0.3)
    np.savez_compressed(OUT / "golden_detect.npz", **d)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
