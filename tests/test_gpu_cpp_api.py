"""GPU: the C++ operator API (include/kcache/*.hpp) compiled as a client
program, the way the reference's Engine and tests use it."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_cpp_test():
    exe = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")
    src = exe + ".cpp"
    lib = os.path.join(ROOT, "paper_2404_18057_b200", "libkcache_b200.so")
    if not os.path.exists(exe) or os.path.getmtime(exe) < max(os.path.getmtime(src), os.path.getmtime(lib)):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), src,
                        "-L" + os.path.dirname(lib), "-lkcache_b200",
                        "-Wl,-rpath,$ORIGIN/../../paper_2404_18057_b200", "-o", exe], check=True)
    return exe


def test_cpp_operator_api_cases():
    exe = build_cpp_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
