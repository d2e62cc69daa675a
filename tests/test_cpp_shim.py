"""The C++ drop-in header (include/flashrnn/engine.hpp) used like rnnkit's API.

CPU: the shim and the test program compile against the public headers.
GPU: the program runs forward/backward through the shim for every variant in
fp32 and bf16 and checks the reference's exception behaviour.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
EXE = os.path.join(ROOT, "build", "shim_test")
CUDA = "/usr/local/cuda"


def _flags():
    return ["-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{CUDA}/include"]


def test_shim_compiles():
    r = subprocess.run(["g++"] + _flags() + ["-fsyntax-only", SRC], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                   check=True)
    lib = os.path.join(ROOT, "paper_2412_07752_b200")
    cmd = (["g++"] + _flags() + [SRC, "-o", EXE, f"-L{lib}", "-lflashrnn", f"-L{ROOT}/oracle", "-loracle",
                                 f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{lib}:{ROOT}/oracle:{CUDA}/lib64"])
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_shim_parity_on_gpu():
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "SHIM_TEST PASS" in r.stdout, r.stdout + r.stderr
