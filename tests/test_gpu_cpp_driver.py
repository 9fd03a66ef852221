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


def test_cpp_mgpu_driver_world1_bitwise(tmp_path):
    """The multi-GPU C++ driver (tools/cpp_driver_mgpu.cpp: one process per GPU, NCCL id
    bootstrapped through a shared directory, dc_comm_attach, DA cycles with the barrier
    exchange and the drifter gather inside the library) at world size 1 on this GPU: rank
    0's members and the forecast statistics are bitwise equal to one context holding the
    ensemble. On a multi-GPU box the same binary runs with world = #GPUs."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    exe = str(tmp_path / "mgpu")
    lib = os.path.join(ROOT, "paper_1910_01031_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["g++", "-std=c++17", "-O2", f"-I{ROOT}/include", f"-I{cuda}/include",
           os.path.join(ROOT, "tools", "cpp_driver_mgpu.cpp"), f"-L{lib}", "-ldriftcast_gpu",
           f"-L{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{cuda}/lib64", "-o", exe]
    subprocess.run(cmd, check=True)
    n_gpu = torch.cuda.device_count()
    for world in sorted({1, n_gpu}):
        out = subprocess.run([exe, str(world), "6", "3", str(tmp_path / f"boot{world}"), "100", "60"],
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "cycle 2: E" in out.stdout
        assert "bitwise equal to one context: yes" in out.stdout
