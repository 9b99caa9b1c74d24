"""The C++ drop-in shim (include/dfftb/dfft.hpp) compiled with reference
test bodies (tests/cpp/test_shim.cpp) and linked against libdfftb.so."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PKG = os.path.join(ROOT, "paper_1506_07933_b200")
BIN = os.path.join(HERE, "cpp", "test_shim")


def _build():
    src = os.path.join(HERE, "cpp", "test_shim.cpp")
    if os.path.exists(BIN) and os.path.getmtime(BIN) > max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(ROOT, "include", "dfftb", "dfft.hpp")),
            os.path.getmtime(os.path.join(ROOT, "include", "dfftb", "tensor_file.hpp")),
            os.path.getmtime(os.path.join(PKG, "libdfftb.so"))):
        return
    cmd = ["g++", "-std=c++20", "-O1", "-o", BIN, src, "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", "-L", PKG, "-ldfftb", f"-Wl,-rpath,{PKG}",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)


def test_shim_host_side():
    _build()
    r = subprocess.run([BIN, "--host"], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0


@pytest.mark.gpu
def test_shim_execute_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0
