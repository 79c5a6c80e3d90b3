"""The C++ drop-in entry point: a small C++ program (tests/cpp/) compiled
against include/ and linked with libdapple.so plans, simulates and then
executes one step with pipeplan::execute_plan on cuda:0."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(ROOT, "paper_2007_01045_b200")


@pytest.mark.skipif(not shutil.which("g++"), reason="g++ not available")
def test_cpp_execute_plan(cuda, tmp_path):
    exe = tmp_path / "demo"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", os.path.join(HERE, "cpp", "execute_plan_demo.cpp"),
                    "-o", str(exe), f"-L{LIB_DIR}", "-ldapple", f"-Wl,-rpath,{LIB_DIR}"], check=True,
                   capture_output=True, text=True, timeout=300)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.startswith("stages ")
