"""CPU tests of the boundary: the C-ABI library loads, exports every symbol
include/trigraph_b200.h declares (and the Python mirror binds them all), the
C++ mirror header compiles and links against it, host-side validation
raises the reference's exception types, and -- without a GPU -- compute
entry points fail loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1706_05151_b200 import _lib
from paper_1706_05151_b200 import trigraph as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "trigraph_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 30
    L = C.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), f"{s} declared in trigraph_b200.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(syms)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_cpp_mirror_compiles_and_links(tmp_path):
    exe = tmp_path / "parity_main"
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "parity_main.cpp"), "-o", str(exe),
           _lib.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cpp_comm_driver_compiles_and_links(tmp_path):
    exe = tmp_path / "comm_main"
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
           "/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "comm_main.cpp"), "-o",
           str(exe), _lib.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_host_validation_maps_to_reference_exceptions():
    with pytest.raises(ValueError):
        T._cfg(T.EngineConfig(engine=T.EngineKind.Aop, ranks=2, boundaries=[0, 1]))
    with pytest.raises(ValueError):
        T._cfg(T.EngineConfig(order="alphabetical"))  # cli.hpp:67-72 unknown ordering
    c, _ = T._cfg(T.EngineConfig(order=T.OrderKind.by_random(9)))
    assert (c.order_set, c.order, c.order_seed) == (1, int(T.OrderTag.ByRandom), 9)
    c, _ = T._cfg(T.EngineConfig(order="coreness"))
    assert (c.order, c.order_seed) == (int(T.OrderTag.ByCoreness), 0)
    assert T.EngineConfig().order == T.OrderKind.by_degree()  # engines.hpp:274
    assert T.to_string(T.EngineKind.AnopSurrogate) == "anop-surrogate"
    assert T.to_string(T.CostKind.Dpd) == "DPD"
    plan = T.PartitionPlan(np.array([0, 2, 2, 5, 7], np.uint32))  # test_partition.cpp:97-107
    assert [plan.owner(v) for v in range(7)] == [0, 0, 2, 2, 2, 3, 3]
    assert all(plan.in_core(plan.owner(v), v) for v in range(7))


def test_generator_argument_errors():
    with pytest.raises(ValueError):
        T.gen_pa(10, 3, 1)  # io.hpp:130-131: d must be even
    with pytest.raises(ValueError):
        T.gen_gnp(10, 20.0, 1)
    with pytest.raises(ValueError):
        T.gen_ws(10, 3, 0.1, 1)


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises((_lib.TrigraphError, ValueError)):
        T.build_graph([(0, 1), (1, 2), (0, 2)])


def test_stats_helpers():
    # stats.hpp:11-23; acceptance.cpp:469-476 (p_opt extrapolation: 120 * sqrt(25) = 600)
    assert T.estimate_p_opt(25e6, 50, 1e6, 50, 120) == 600
    assert T.estimate_p_opt(1e6, 100, 1e6, 50, 3) == 6
    with pytest.raises(ValueError):
        T.estimate_p_opt(0, 50, 1e6, 50, 120)
    assert T.normalized_triangle_count(10, 4) == 2.5
    assert T.normalized_triangle_count(10, 0) == 0.0
