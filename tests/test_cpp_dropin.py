"""The pardyn drop-in C++ API (include/pardyn/pardyn.hpp, libpardyn.so over
the C-ABI): compiled and linked on CPU; run on the GPU as a C++ program that
reads like the reference's test_fwddyn.cpp (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1609_06779_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    cmd = ["g++", "-O2", "-std=c++20", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           "-o", exe, f"-L{LIB}", "-lpardyn", "-lpardyn_b200", f"-Wl,-rpath,{LIB}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    assert os.path.exists(os.path.join(LIB, "libpardyn.so"))
    build(tmp_path)


def test_dropin_without_gpu_fails_loudly(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert r.returncode != 0 and "cannot open CUDA device" in r.stderr


@pytest.mark.gpu
def test_dropin_cpp_suite_on_gpu(tmp_path):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout
