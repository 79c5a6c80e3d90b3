"""Drop-in check of the C++ boundary: the reference's own acceptance program
(proj/tests/acceptance.cpp + its harness.cpp, compiled from /root/reference)
built against *this* repo's include/pipeplan headers and linked with
libdapple.so must print exactly what the reference-built binary prints.
CPU only; skipped where /root/reference or the oracle build is absent."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = "/root/reference/proj"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance")
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
LIB_DIR = os.path.join(ROOT, "paper_2007_01045_b200")


@pytest.mark.skipif(not (os.path.isdir(REF) and os.path.exists(REF_BIN) and shutil.which("g++")
                         and os.path.isdir(NLOHMANN)), reason="reference sources / oracle build not available")
def test_reference_acceptance_runs_unchanged_on_this_library(tmp_path):
    exe = tmp_path / "acceptance_ours"
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-w",
           f"-I{ROOT}/include",            # our pipeplan headers first ...
           f"-I{REF}/include",             # ... the reference only for harness.hpp
           f"-I{NLOHMANN}", f"-I{REF}/tests",
           f"{REF}/tests/acceptance.cpp", f"{REF}/src/harness.cpp", "-o", str(exe),
           f"-L{LIB_DIR}", "-ldapple", f"-Wl,-rpath,{LIB_DIR}", "-lpthread"]
    subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=600)
    ours = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900).stdout
    ref = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=900).stdout
    assert ours == ref
    assert "of 7 criteria passed" in ours
