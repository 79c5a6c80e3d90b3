"""Client for oracle/_ref/ref_cli (TEST INFRASTRUCTURE ONLY).

Spawns the compiled reference once and sends it JSON requests
(see oracle/ref_bridge.cpp for the vocabulary).
"""
import json
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_CLI = os.path.join(_HERE, "_ref", "ref_cli")


class ReferenceProcess:
    def __init__(self, path=REF_CLI):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (needs /root/reference)")
        self._p = subprocess.Popen([path], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True, bufsize=1)
        self._lock = threading.Lock()

    def call(self, request: dict) -> dict:
        with self._lock:
            self._p.stdin.write(json.dumps(request) + "\n")
            self._p.stdin.flush()
            line = self._p.stdout.readline()
        if not line:
            raise RuntimeError("reference oracle process exited")
        return json.loads(line)

    def close(self):
        try:
            self._p.stdin.close()
            self._p.wait(timeout=5)
        except Exception:
            self._p.kill()


_shared = None


def shared() -> ReferenceProcess:
    global _shared
    if _shared is None:
        _shared = ReferenceProcess()
    return _shared


def available() -> bool:
    return os.path.exists(REF_CLI)
