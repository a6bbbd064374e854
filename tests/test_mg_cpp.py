"""A C++ caller of the multi-GPU C ABI (tests/cpp/mg_nccl.cpp): gbx_comm_init
over NCCL (one rank), the distributed build and every gbx_*_mg call against the
oracle.  The build runs on CPU (it only links); the run needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "oracle", "_build", "mg_nccl")


def build():
    import oracle
    oracle.build(ref=False)
    cmd = ["g++", "-std=c++17", "-O1", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "mg_nccl.cpp"), "-o", OUT,
           f"-L{ROOT}/oracle/_build", "-lorc", f"-L{ROOT}/paper_2104_01661_b200", "-lgbx",
           f"-Wl,-rpath,{ROOT}/oracle/_build", f"-Wl,-rpath,{ROOT}/paper_2104_01661_b200"]
    subprocess.run(cmd, check=True)
    return OUT


def test_mg_cpp_caller_builds():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_mg_cpp_caller_runs_over_nccl():
    exe = OUT if os.path.exists(OUT) else build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mg nccl ok" in r.stdout
