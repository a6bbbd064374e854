"""The C++ drop-in adapter (include/gbx_gblite.hpp) compiles against the
reference's headers and links against libgbx.so + the reference library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
OUT = os.path.join(ROOT, "oracle", "_ref", "adapter_smoke")


def build_adapter():
    import oracle
    oracle.build(ref=True)
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", f"-I{REF}/include",
           os.path.join(ROOT, "tests", "cpp", "adapter_smoke.cpp"), "-o", OUT,
           f"-L{ROOT}/oracle/_ref", "-lgblite_ref", f"-L{ROOT}/paper_2104_01661_b200", "-lgbx",
           f"-Wl,-rpath,{ROOT}/oracle/_ref", f"-Wl,-rpath,{ROOT}/paper_2104_01661_b200"]
    subprocess.run(cmd, check=True)
    return OUT


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference headers not present")
def test_adapter_compiles_and_links():
    exe = build_adapter()
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    assert "adapter linked" in out


@pytest.mark.gpu
def test_adapter_runs_against_reference():
    exe = OUT
    if not os.path.exists(exe):
        pytest.skip("adapter binary not built (needs the reference headers at build time)")
    r = subprocess.run([exe, "run"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
