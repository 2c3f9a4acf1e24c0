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
