"""The C++ host side (include/driftcast_gpu.hpp over the C ABI) builds with g++ and runs
DA cycles on the GPU; exceptions map back to the reference types."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_cpp_driver_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    exe = str(tmp_path / "driver")
    lib = os.path.join(ROOT, "paper_1910_01031_b200")
    cmd = ["g++", "-std=c++17", "-O2", f"-I{ROOT}/include",
           os.path.join(ROOT, "tools", "cpp_driver_example.cpp"), f"-L{lib}", "-ldriftcast_gpu",
           f"-Wl,-rpath,{lib}", "-o", exe]
    subprocess.run(cmd, check=True)
    out = subprocess.run([exe, "8", "2", str(tmp_path / "ck")], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    assert "cycle 1:" in out.stdout and "invalid_argument caught" in out.stdout
    assert "t = 600.0 s" in out.stdout
    assert "restart from checkpoint reproduces the run: yes" in out.stdout
    assert "max PF log-likelihood" in out.stdout
