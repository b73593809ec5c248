"""The C++ drop-in (include/adattn_b200/attention.hpp) built against
libadattn_b200.so and run through the reference's own test_attention.cpp
scenarios (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_reference_scenarios(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2604_15180_b200")
    exe = str(tmp_path / "test_shim")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L", lib_dir,
                    "-ladattn_b200", f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
