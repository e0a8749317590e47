"""The C-ABI used from plain C (examples/abi_demo.c: no Python, no torch): host-memory sketch
(Alg. 1), self-join (Def. 6), ranking (Alg. 2) and a brute-force check of the top discord."""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_demo_runs(cuda, tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib = os.path.join(ROOT, "paper_2311_03393_b200")
    exe = str(tmp_path / "abi_demo")
    r = subprocess.run(["gcc", "-std=c99", "-O2", os.path.join(ROOT, "examples", "abi_demo.c"),
                        f"-I{os.path.join(ROOT, 'include')}", "-I/usr/local/cuda/include", f"-L{lib}", "-lsketchmp",
                        "-L/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{lib}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "abi_demo ok" in out.stdout, out.stdout + out.stderr
