"""Build the C++ host-API test program (tests/cpp/test_host_api.cpp) against
libstg_cuda.so -- compile check on CPU, run on the GPU."""
import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_host_api.cpp"
LIBDIR = ROOT / "paper_2201_05800_b200"


def _build(tmp_path: Path) -> Path:
    from paper_2201_05800_b200 import build as B
    B.build()
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")
    exe = tmp_path / "test_host_api"
    cmd = [cxx, "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(SRC),
           f"-L{LIBDIR}", "-lstg_cuda", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_host_api_compiles(tmp_path):
    exe = _build(tmp_path)
    assert exe.exists()


def test_cpp_host_field_helpers_run_on_cpu(tmp_path):
    """node_coord / interpolate / global_mass / l2_error of the C++ mirror
    (test_mesh.cpp:70-190 ported): host-only, no device."""
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), "--host-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed 0" in r.stdout


@pytest.mark.gpu
def test_cpp_host_api_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed 0" in r.stdout


@pytest.mark.parametrize("threads", ["1", "3", "8"])
def test_host_copy_pool_equals_memcpy(tmp_path, threads):
    """The worker-thread copies behind pageable host buffers
    (csrc/hostcopy.hpp): ragged multi-item copies equal memcpy."""
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")
    exe = tmp_path / "test_hostcopy"
    subprocess.run([cxx, "-std=c++17", "-O2", "-Wall", "-Wextra", "-pthread",
                    str(ROOT / "tests" / "cpp" / "test_hostcopy.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120,
                       env={**os.environ, "STG_HOST_THREADS": threads})
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"threads {threads} failed 0" in r.stdout
