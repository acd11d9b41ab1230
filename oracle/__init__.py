"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the hsad hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and the CPU-baseline legs of
``bench.py`` may import this package, and only as the checker / the timed CPU
baseline, never as the product. Two libraries are exposed:

* ``port``  — ``oracle/_build/libhsad_oracle.so``: the Eigen-free C++
  restatement of proj/core/src/{wavelet,stats,detect}.cpp (hsad_oracle.cpp);
* ``ref``   — ``oracle/_ref/libhsad_ref.so``: the reference's own Eigen-free
  translation units (wavelet.cpp, error.cpp, tests/support/oracles.cpp)
  compiled in place by oracle/Makefile. ``None`` when it was not built.

Both are plain ctypes bindings over numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "_build" / "libhsad_oracle.so"
REF_SO = HERE / "_ref" / "libhsad_ref.so"

ERRC_NAMES = [
    "Ok", "MissingKey", "InvalidValue", "SizeMismatch", "NonFiniteValue", "OutOfBounds",
    "UnsupportedOrder", "OddLength", "TooShort", "LengthMismatch", "TargetTooLarge",
    "EmptySampleSet", "TooFewSamples", "SingularAfterRidge", "NotSymmetric", "NoConvergence",
    "ConfigMismatch", "FractionOutOfRange", "OutOfBoundsImplant", "DimensionMismatch",
    "DegenerateTruth", "IoFailure",
]


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str, row: int = -1, col: int = -1):
        super().__init__(message)
        self.code = code
        self.name = ERRC_NAMES[code] if 0 <= code < len(ERRC_NAMES) else "Unknown"
        self.row, self.col = row, col


def build() -> None:
    """Compile the restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _load(path: Path):
    return C.CDLL(str(path)) if path.exists() else None


_D = C.POINTER(C.c_double)
_I8 = C.POINTER(C.c_int8)
_L = C.POINTER(C.c_long)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _vp(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class _Port:
    def __init__(self, lib):
        self.lib = lib
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_random_cube.argtypes = [C.c_long, C.c_long, C.c_int, C.c_uint64, C.c_double,
                                        C.c_double, _D]
        lib.orc_random_signal.argtypes = [C.c_long, C.c_uint64, C.c_double, C.c_double, _D]
        lib.orc_mirror_index.argtypes = [C.c_int, C.c_int]
        V, I, Lg, Dd = C.c_void_p, C.c_int, C.c_long, C.c_double
        P = C.POINTER
        lib.orc_daubechies.argtypes = [I, _D, _D, P(C.c_int)]
        lib.orc_dwt_level.argtypes = [_D, I, I, _D, _D]
        lib.orc_idwt_level.argtypes = [_D, _D, I, I, _D]
        lib.orc_multilevel_approx.argtypes = [_D, I, I, I, _D]
        lib.orc_reduce_cube.argtypes = [V, I, Lg, Lg, I, I, I, _D, I]
        lib.orc_window_validate.argtypes = [I, I, I]
        lib.orc_mean_vector.argtypes = [_D, I, I, _D]
        lib.orc_covariance.argtypes = [_D, I, I, _D, _D]
        lib.orc_regularized_inverse.argtypes = [_D, I, Dd, _D, _D]
        lib.orc_symmetric_eigen.argtypes = [_D, I, _D, _D]
        lib.orc_local_rx_rows.argtypes = [V, I, Lg, Lg, I, Lg, Lg, I, I, Dd, _D, I, _L, _L]
        lib.orc_dwrx_rows.argtypes = [V, I, Lg, Lg, I, Lg, Lg, I, I, Dd, _D, I, _L, _L]
        lib.orc_dwest_rows.argtypes = [V, I, Lg, Lg, I, Lg, Lg, I, I, Dd, _D, _I8, I, _L, _L]
        lib.orc_dwest_margins.argtypes = [V, I, Lg, Lg, I, Lg, Lg, I, I, Dd, _D, _D, I]
        lib.orc_hp_lrx_pixels.argtypes = [V, I, Lg, Lg, I, I, I, Dd, Lg, _L, _L, _D, _D, I]
        lib.orc_hp_dwrx_pixels.argtypes = [V, I, Lg, Lg, I, I, I, Dd, Lg, _L, _L, _D, _D, I]

    def _check(self, rc: int, row: int = -1, col: int = -1):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode(), row, col)

    # --- RNG of proj/tests/support/testutil.hpp -----------------------------
    def random_cube(self, lines, samples, bands, seed, lo=0.0, hi=1.0) -> np.ndarray:
        out = np.empty((lines, samples, bands), np.float64)
        self.lib.orc_random_cube(lines, samples, bands, seed, lo, hi, _dp(out))
        return out

    def random_signal(self, length, seed, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(length, np.float64)
        self.lib.orc_random_signal(length, seed, lo, hi, _dp(out))
        return out

    # --- wavelet ----------------------------------------------------------------
    def daubechies(self, order):
        low = np.zeros(32); high = np.zeros(32); n = C.c_int(0)
        self._check(self.lib.orc_daubechies(order, _dp(low), _dp(high), C.byref(n)))
        return low[: n.value].copy(), high[: n.value].copy()

    def dwt_level(self, x, order):
        x = np.ascontiguousarray(x, np.float64)
        a = np.zeros(max(len(x) // 2, 1)); d = np.zeros(max(len(x) // 2, 1))
        self._check(self.lib.orc_dwt_level(_dp(x), len(x), order, _dp(a), _dp(d)))
        return a[: len(x) // 2], d[: len(x) // 2]

    def idwt_level(self, a, d, order):
        a = np.ascontiguousarray(a, np.float64); d = np.ascontiguousarray(d, np.float64)
        out = np.zeros(2 * len(a))
        self._check(self.lib.orc_idwt_level(_dp(a), _dp(d), len(a), order, _dp(out)))
        return out

    def multilevel_approx(self, x, order, target):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(max(target, 1) * 2 + len(x))
        self._check(self.lib.orc_multilevel_approx(_dp(x), len(x), order, target, _dp(out)))
        return out[:target].copy()

    def reduce_cube(self, cube: np.ndarray, order=2, target=4, workers=1) -> np.ndarray:
        cube = np.ascontiguousarray(cube)
        assert cube.dtype in (np.float32, np.float64)
        lines, samples, bands = cube.shape
        out = np.zeros((lines, samples, target), np.float64)
        self._check(self.lib.orc_reduce_cube(_vp(cube), cube.dtype.itemsize, lines, samples,
                                             bands, order, target, _dp(out), workers))
        return out

    # --- geometry / stats -----------------------------------------------------
    def mirror_index(self, i, n):
        return self.lib.orc_mirror_index(i, n)

    def window_validate(self, mode, a, b=0):
        self._check(self.lib.orc_window_validate(mode, a, b))

    def mean_vector(self, samples):  # samples: (count, dim)
        s = np.ascontiguousarray(samples, np.float64)
        out = np.zeros(s.shape[1] if s.ndim == 2 else 0)
        self._check(self.lib.orc_mean_vector(_dp(s), s.shape[1], s.shape[0], _dp(out)))
        return out

    def covariance(self, samples, mean=None):
        s = np.ascontiguousarray(samples, np.float64)
        mean = self.mean_vector(s) if mean is None else np.ascontiguousarray(mean, np.float64)
        out = np.zeros((s.shape[1], s.shape[1]))
        self._check(self.lib.orc_covariance(_dp(s), s.shape[1], s.shape[0], _dp(mean), _dp(out)))
        return out

    def regularized_inverse(self, cov, ridge):
        c = np.ascontiguousarray(cov, np.float64)
        out = np.zeros_like(c); applied = C.c_double(0)
        self._check(self.lib.orc_regularized_inverse(_dp(c), c.shape[0], ridge, _dp(out),
                                                     C.byref(applied)))
        return out, applied.value

    def symmetric_eigen(self, m):
        m = np.ascontiguousarray(m, np.float64)
        n = m.shape[0]
        vals = np.zeros(n); vecs = np.zeros((n, n))
        # column-major in C: vecs[i] (row of the numpy array) is eigenvector i
        self._check(self.lib.orc_symmetric_eigen(_dp(np.asfortranarray(m).T.copy()), n,
                                                 _dp(vals), _dp(vecs)))
        return vals, vecs.T.copy()  # columns are eigenvectors

    # --- detectors --------------------------------------------------------------
    def _cube(self, cube):
        cube = np.ascontiguousarray(cube)
        if cube.dtype not in (np.float32, np.float64):
            cube = cube.astype(np.float64)
        return cube

    def local_rx(self, cube, window, ridge=1e-6, guard=1, workers=1, rows=None):
        cube = self._cube(cube); L, S, B = cube.shape
        rb, re = rows if rows else (0, L)
        out = np.zeros((re - rb, S)); er = C.c_long(-1); ec = C.c_long(-1)
        rc = self.lib.orc_local_rx_rows(_vp(cube), cube.dtype.itemsize, L, S, B, rb, re, window,
                                        guard, C.c_double(ridge), _dp(out), workers,
                                        C.byref(er), C.byref(ec))
        self._check(rc, er.value, ec.value)
        return out

    def dwrx(self, cube, inner, outer, ridge=1e-6, workers=1, rows=None):
        cube = self._cube(cube); L, S, B = cube.shape
        rb, re = rows if rows else (0, L)
        out = np.zeros((re - rb, S)); er = C.c_long(-1); ec = C.c_long(-1)
        rc = self.lib.orc_dwrx_rows(_vp(cube), cube.dtype.itemsize, L, S, B, rb, re, inner, outer,
                                    C.c_double(ridge), _dp(out), workers, C.byref(er), C.byref(ec))
        self._check(rc, er.value, ec.value)
        return out

    def dwest(self, cube, inner, outer, eigen_fraction=0.1, workers=1, rows=None):
        cube = self._cube(cube); L, S, B = cube.shape
        rb, re = rows if rows else (0, L)
        out = np.zeros((re - rb, S)); cnt = np.zeros((re - rb, S), np.int8)
        er = C.c_long(-1); ec = C.c_long(-1)
        rc = self.lib.orc_dwest_rows(_vp(cube), cube.dtype.itemsize, L, S, B, rb, re, inner,
                                     outer, C.c_double(eigen_fraction), _dp(out),
                                     cnt.ctypes.data_as(_I8), workers, C.byref(er), C.byref(ec))
        self._check(rc, er.value, ec.value)
        return out, cnt

    # --- extended-precision third opinion (hp_oracle.cpp) ------------------------
    def _hp(self, fn, cube, a, b, ridge, rows, cols, workers):
        cube = self._cube(cube); L, S, B = cube.shape
        rows = np.ascontiguousarray(rows, np.int64); cols = np.ascontiguousarray(cols, np.int64)
        out = np.zeros(len(rows)); piv = np.zeros(len(rows))
        fn(_vp(cube), cube.dtype.itemsize, L, S, B, a, b, C.c_double(ridge), len(rows),
           rows.ctypes.data_as(_L), cols.ctypes.data_as(_L), _dp(out), _dp(piv), workers)
        return out, piv

    def hp_local_rx(self, cube, window, rows, cols, ridge=1e-6, guard=1, workers=1):
        """LRX in long double at the listed pixels: (scores, LDL^T pivot ratio)."""
        return self._hp(self.lib.orc_hp_lrx_pixels, cube, window, guard, ridge, rows, cols, workers)

    def hp_dwrx(self, cube, inner, outer, rows, cols, ridge=1e-6, workers=1):
        return self._hp(self.lib.orc_hp_dwrx_pixels, cube, inner, outer, ridge, rows, cols, workers)

    def dwest_margins(self, cube, inner, outer, eigen_fraction=0.1, workers=1, rows=None):
        cube = self._cube(cube); L, S, B = cube.shape
        rb, re = rows if rows else (0, L)
        cm = np.zeros((re - rb, S)); sm = np.zeros((re - rb, S))
        self._check(self.lib.orc_dwest_margins(_vp(cube), cube.dtype.itemsize, L, S, B, rb, re,
                                               inner, outer, C.c_double(eigen_fraction), _dp(cm),
                                               _dp(sm), workers))
        return cm, sm


class _Ref:
    """The reference's own sources (wavelet.cpp + tests/support/oracles.cpp)."""

    def __init__(self, lib):
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        I, Dd = C.c_int, C.c_double
        lib.ref_daubechies.argtypes = [I, _D, _D, C.POINTER(C.c_int)]
        lib.ref_dwt_level.argtypes = [_D, I, I, _D, _D]
        lib.ref_idwt_level.argtypes = [_D, _D, I, I, _D]
        lib.ref_multilevel_approx.argtypes = [_D, I, I, I, _D]
        lib.ref_reduce_cube.argtypes = [_D, I, I, I, I, I, _D, I]
        lib.ref_brute_dwt.argtypes = [_D, I, I, _D, _D]
        lib.ref_brute_covariance.argtypes = [_D, I, I, _D]
        lib.ref_jacobi_eigen.argtypes = [_D, I, _D, _D]
        lib.ref_naive_lrx.argtypes = [_D, I, I, I, I, Dd, _D]
        lib.ref_naive_dwrx.argtypes = [_D, I, I, I, I, I, Dd, _D]
        lib.ref_naive_dwest.argtypes = [_D, I, I, I, I, I, Dd, _D]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def daubechies(self, order):
        low = np.zeros(32); high = np.zeros(32); n = C.c_int(0)
        self._check(self.lib.ref_daubechies(order, _dp(low), _dp(high), C.byref(n)))
        return low[: n.value].copy(), high[: n.value].copy()

    def dwt_level(self, x, order):
        x = np.ascontiguousarray(x, np.float64)
        a = np.zeros(max(len(x) // 2, 1)); d = np.zeros(max(len(x) // 2, 1))
        self._check(self.lib.ref_dwt_level(_dp(x), len(x), order, _dp(a), _dp(d)))
        return a[: len(x) // 2], d[: len(x) // 2]

    def idwt_level(self, a, d, order):
        a = np.ascontiguousarray(a, np.float64); d = np.ascontiguousarray(d, np.float64)
        out = np.zeros(2 * len(a))
        self._check(self.lib.ref_idwt_level(_dp(a), _dp(d), len(a), order, _dp(out)))
        return out

    def multilevel_approx(self, x, order, target):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(max(target, 1) * 2 + len(x))
        self._check(self.lib.ref_multilevel_approx(_dp(x), len(x), order, target, _dp(out)))
        return out[:target].copy()

    def reduce_cube(self, cube, order=2, target=4, workers=1):
        cube = np.ascontiguousarray(cube, np.float64)
        L, S, B = cube.shape
        out = np.zeros((L, S, target))
        self._check(self.lib.ref_reduce_cube(_dp(cube), L, S, B, order, target, _dp(out), workers))
        return out

    def brute_dwt(self, x, order):
        x = np.ascontiguousarray(x, np.float64)
        a = np.zeros(len(x) // 2); d = np.zeros(len(x) // 2)
        self.lib.ref_brute_dwt(_dp(x), len(x), order, _dp(a), _dp(d))
        return a, d

    def brute_covariance(self, samples):  # (count, dim)
        s = np.ascontiguousarray(samples, np.float64)
        out = np.zeros((s.shape[1], s.shape[1]))
        self.lib.ref_brute_covariance(_dp(s), s.shape[1], s.shape[0], _dp(out))
        return out

    def jacobi_eigen(self, m):
        m = np.ascontiguousarray(m, np.float64)
        n = m.shape[0]
        vals = np.zeros(n); vecs = np.zeros((n, n))
        self.lib.ref_jacobi_eigen(_dp(m), n, _dp(vals), _dp(vecs))
        return vals, vecs

    def naive_lrx(self, cube, window, ridge):
        cube = np.ascontiguousarray(cube, np.float64); L, S, B = cube.shape
        out = np.zeros((L, S))
        self.lib.ref_naive_lrx(_dp(cube), L, S, B, window, C.c_double(ridge), _dp(out))
        return out

    def naive_dwrx(self, cube, inner, outer, ridge):
        cube = np.ascontiguousarray(cube, np.float64); L, S, B = cube.shape
        out = np.zeros((L, S))
        self.lib.ref_naive_dwrx(_dp(cube), L, S, B, inner, outer, C.c_double(ridge), _dp(out))
        return out

    def naive_dwest(self, cube, inner, outer, frac):
        cube = np.ascontiguousarray(cube, np.float64); L, S, B = cube.shape
        out = np.zeros((L, S))
        self.lib.ref_naive_dwest(_dp(cube), L, S, B, inner, outer, C.c_double(frac), _dp(out))
        return out


if not PORT_SO.exists() and os.environ.get("HSAD_ORACLE_NO_BUILD") != "1":
    try:
        build()
    except Exception:  # pragma: no cover - surfaced by the tests that need it
        pass

port = _Port(_load(PORT_SO)) if PORT_SO.exists() else None
ref = _Ref(_load(REF_SO)) if REF_SO.exists() else None


def rel_diff(a, b):
    """|a-b| / max(1, |a|, |b|) — proj/tests/support/testutil.hpp:34-36."""
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def max_rel_diff(a, b) -> float:
    d = rel_diff(a, b)
    return float(d.max()) if d.size else 0.0
