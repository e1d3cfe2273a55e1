"""The header-only C++ facade (include/hmat_b200.hpp) compiles reference-style client
code and links against libhmat_b200.so; on a GPU the demo also runs end to end."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(REPO, "tests", "cpp", "facade_demo.cpp")
LIBDIR = os.path.join(REPO, "paper_1708_09707_b200")


def build(tmp_path):
    exe = str(tmp_path / "facade_demo")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(REPO, "include"), SRC, "-o", exe, "-L", LIBDIR,
                    "-lhmat_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_facade_runs_on_gpu(tmp_path, gpu):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok" in out.stdout
