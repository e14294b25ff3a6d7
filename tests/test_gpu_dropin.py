"""The C++ drop-in API (include/dedisp/b200.hpp) compiled like reference
client code and run on the GPU (tests/cxx/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_cxx_dropin(tmp_path, golden):
    from oracle import oracle as O
    from paper_1601_05052_b200 import api
    if api.device_count() == 0:
        pytest.skip("no CUDA device")
    O.lib()  # builds oracle/liboracle.so when needed
    pkg = os.path.join(ROOT, "paper_1601_05052_b200")
    exe = str(tmp_path / "dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cxx", "test_dropin.cpp"), "-L", pkg,
                    "-ldedisp_b200", "-L", os.path.join(ROOT, "oracle"), "-loracle",
                    f"-Wl,-rpath,{pkg}:{os.path.join(ROOT, 'oracle')}", "-o", exe], check=True)
    g4k = [b for b in golden["baseline"]
           if b["setup"]["name"] == "Apertif" and b["num_dms"] == 4096][0]["out_fnv"]
    r = subprocess.run([exe, g4k], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin: ok" in r.stdout
    assert f"fingerprint {g4k}" in r.stdout
