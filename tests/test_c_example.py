"""The C ABI from plain C (examples/dgemm_c.c): the header compiles as C11 with warnings as
errors and the program links against liboz2.so alone (no Python, no torch).  On a GPU the
program runs an emulated DGEMM on host buffers and checks it against a long-double triple
loop; without one it must fail loudly (non-zero exit), never fall back to the CPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2603_10634_b200")


def _build(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "liboz2.so")):
        pytest.skip("liboz2.so not built")
    exe = str(tmp_path / "dgemm_c")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "dgemm_c.c"), "-L", LIBDIR, "-loz2", f"-Wl,-rpath,{LIBDIR}", "-lm",
           "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_builds_and_fails_loudly_without_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "64", "64", "64", "13"], capture_output=True, text=True, timeout=300)
    assert "oz2 " in r.stdout and "sm_100a" in r.stdout
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert r.returncode != 0 and "oz2_dgemm returned" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [("300", "200", "250", "13"), ("600", "2000", "500", "14")])
def test_c_example_runs_on_gpu(tmp_path, shape):
    exe = _build(tmp_path)
    r = subprocess.run([exe, *shape], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "status=0" in r.stdout
