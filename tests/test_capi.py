"""The C-ABI library loads without a GPU and exports every symbol that
include/dapple.h declares; host entry points work on CPU."""
import ctypes
import json
import os
import re

from paper_2007_01045_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dapple.h")).read()
    return sorted(set(re.findall(r"\b(dpl_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.exported_symbols()) | {"dpl_version"}


def test_cpp_api_symbols_exported():
    import subprocess
    out = subprocess.run(["nm", "-DC", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for fn in ["pipeplan::plan(", "pipeplan::simulate_plan(", "pipeplan::execute_plan(", "pipeplan::dapple_schedule(",
               "pipeplan::estimate_latency(", "pipeplan::load_profile(", "pipeplan::plan_from_json(",
               "pipeplan::splitconcat_routes(", "pipeplan::write_timeline_csv("]:
        assert fn in out, fn


def test_host_call_and_errors():
    lib = _lib.lib()
    r = json.loads(lib.dpl_host_call(b'{"op": "expand_plan_phi", "phi": [2, 1]}'))
    assert r == {"phi": [2, 1, 1]}
    r = json.loads(lib.dpl_host_call(b'{"op": "nope"}'))
    assert r["error"]["type"] == "invalid_argument"
    r = json.loads(lib.dpl_host_call(b"not json"))
    assert r["error"]["type"] == "runtime_error"
    assert lib.dpl_version().startswith(b"dapple-b200")


def test_executor_create_fails_cleanly_without_gpu_or_bad_plan():
    import torch
    if torch.cuda.is_available():
        return
    lib = _lib.lib()
    h = ctypes.c_void_p()
    cfg = {"model": {"kind": "mlp", "layers": 2, "hidden": 64}, "plan": {"stages": [{"layers": [0, 2], "gpus": [0]}]},
           "M": 2, "gbs": 4}
    rc = lib.dpl_exec_create(json.dumps(cfg).encode(), 0, ctypes.byref(h))
    assert rc != 0 and lib.dpl_last_error()
