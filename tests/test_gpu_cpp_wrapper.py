"""The C++ drop-in (include/scout_b200.hpp) against the reference's own unit
test cases, restated in tests/cpp/test_wrapper.cpp: compiled here with nvcc,
linked to libscout_b200.so, run on the GPU."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_dropin_passes_reference_cases(cuda, tmp_path):
    exe = tmp_path / "test_wrapper"
    lib = ROOT / "paper_2603_27138_b200"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++20", "-O2", "-Wno-deprecated-gpu-targets", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "test_wrapper.cpp"), "-o", str(exe), "-L", str(lib),
                    "-lscout_b200", f"-Xlinker=-rpath={lib}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout + r.stderr
