"""The C++ drop-in shim (tests/shim/hpeel_shim.hpp): reference-style code --
a LinearOperator subclass, BoxTree::build, compress(op, tree, cfg) ->
PeelResult -- compiled against include/hpeel_b200.h and libhpeel_b200.so.
CPU: it compiles and links. GPU: the host-pointer callback (the reference's
call pattern) and the device-pointer callback (cuBLAS on the driver's
stream) reproduce the built-in dense black box, with the reference's column
counts and exception types."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2205_03406_b200")
SHIM = os.path.join(ROOT, "tests", "shim")


def _build_host(tmp_path):
    exe = str(tmp_path / "shim_main")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(SHIM, "shim_main.cpp"), "-L" + PKG, "-l:libhpeel_b200.so",
                    "-Wl,-rpath," + PKG, "-o", exe], check=True)
    return exe


def _build_device(tmp_path):
    exe = str(tmp_path / "shim_device")
    subprocess.run(["nvcc", "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", "-I",
                    os.path.join(ROOT, "include"), os.path.join(SHIM, "shim_device.cu"), "-L" + PKG,
                    "-l:libhpeel_b200.so", "-lcublas", "-Xlinker", "-rpath," + PKG, "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(_build_host(tmp_path))
    if shutil.which("nvcc"):
        assert os.path.exists(_build_device(tmp_path))


@pytest.mark.gpu
def test_shim_host_callback(tmp_path, gpu_available):
    out = subprocess.run([_build_host(tmp_path), "1024"], check=True, capture_output=True, text=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    # CountingOperator columns == the report's (proj/src/operators.cpp:320-342)
    assert r["counted_forward_cols"] == r["report_forward_cols"] > 0
    assert r["counted_adjoint_cols"] == r["report_adjoint_cols"] > 0
    assert r["rel_error"] < 1e-6, r
    assert r["threw_invalid_argument"]
    assert r["csv_lines"] == r["depth"] + 1  # header + levels 2..depth + leaf


@pytest.mark.gpu
def test_shim_device_callback(tmp_path, gpu_available):
    out = subprocess.run([_build_device(tmp_path), "1024"], check=True, capture_output=True, text=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["device_calls"] > 0
    assert r["dev_vs_host"] < 1e-10 and r["dev_vs_builtin"] < 1e-10, r
    assert r["dev_vs_operator"] < 1e-6 and r["power_method_error"] < 1e-6, r
