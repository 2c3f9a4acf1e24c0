"""Run the reference's own test cases through the C++ mirror on the B200
(tests/cpp/parity_main.cpp: test_sequential.cpp / test_engines.cpp cases
copied unchanged under the namespace alias trigraph = trigraph_b200)."""
import os
import subprocess

import pytest

from paper_1706_05151_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_mirror_runs_reference_cases(tmp_path):
    exe = tmp_path / "parity_main"
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "parity_main.cpp"), "-o", str(exe), _lib.LIB_PATH,
           f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED (0 failures)" in r.stdout


@pytest.mark.parametrize("args", [["3", "local"], ["4", "local"], ["1", "nccl"]])
def test_cpp_host_drives_ranks(tmp_path, args):
    """tests/cpp/comm_main.cpp: one C++ host, a thread per rank, rank-local
    rows, run_engine / AOP step / clustering across ranks through the C ABI
    (csrc/comm.cu) -- the in-process transport with every rank on this box's
    GPU, and NCCL with one rank (an N-GPU node runs `comm_main N nccl`)."""
    exe = tmp_path / "comm_main"
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
           "/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "comm_main.cpp"), "-o",
           str(exe), _lib.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)] + args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED (0 failures)" in r.stdout
