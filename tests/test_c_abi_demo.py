"""The C-ABI used from plain C (examples/c_abi_demo.c): compiles against include/banaserve.h
and links libbanaserve.so with gcc (CPU), and on a B200 migrates a request's blocks
between two pools and checks split attention + merge with q = 0 against the closed form
lse = ln(len), o = mean of the V rows (reading R-A2/R-A3's formulas with every score 0)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2510_13223_b200")


def build_demo(tmp_path) -> str:
    from paper_2510_13223_b200 import build as b
    b.build()
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", os.path.join(ROOT, "examples", "c_abi_demo.c"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + PKG, "-lbanaserve",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-Wl,-rpath," + PKG, "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    assert os.path.exists(build_demo(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs_on_gpu(tmp_path):
    exe = build_demo(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "migrated_bytes_equal=1" in r.stdout
