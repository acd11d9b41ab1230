"""The C++ drop-in (include/hsad/hsad_b200.hpp) compiles against the C-ABI library
on CPU, and its reference-style unit cases pass on the GPU."""
import subprocess
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent / "cpp"


def _build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return HERE / "test_hsad_api"


def test_cpp_dropin_builds():
    assert _build().exists()


@pytest.mark.gpu
def test_cpp_dropin_reference_cases():
    exe = _build()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
