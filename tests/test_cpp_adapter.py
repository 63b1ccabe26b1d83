"""The C++ adapter (include/feti_gpu.hpp) compiles against the C-ABI, links
libfetigpu.so and behaves: host-side construction works without a GPU and
the device build fails loudly there; on a GPU it solves."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2111_11728_b200", "lib")


def _build(tmp_path):
    exe = tmp_path / "adapter_demo"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_demo.cpp"), "-L", LIBDIR,
                    "-lfetigpu", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_adapter_cpu(tmp_path):
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("device present: covered by the gpu test")
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert "dual size" in r.stdout
    assert r.returncode == 2 and "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_adapter_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "solve status 0" in r.stdout
    assert "rebuild + warm solve status 0" in r.stdout
    assert "pivchol rank 2 perm 1 0 L00 2.000250" in r.stdout
