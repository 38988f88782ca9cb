"""TEST INFRASTRUCTURE ONLY: ctypes bridge to oracle/_ref/libsolref.so, the reference solmini
library compiled from /root/reference/proj/src by oracle/Makefile plus oracle/ref_shim.cpp.

Used by tests/, the golden-fixture generator and bench.py's reference/cpu_baseline leg only —
never by the product package. Exposes the reference's f64 oracle (run_reference), its compiled
f32 CPU path and its partition/training-graph builders on graphs given in the reference's own
JSON model schema + SOLW weights.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libsolref.so")
REFERENCE_SRC = "/root/reference/proj/src"

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build(quiet: bool = True) -> bool:
    """Compile the reference (only possible where /root/reference exists)."""
    if not os.path.isdir(REFERENCE_SRC):
        return available()
    import subprocess
    r = subprocess.run(["make", "-C", HERE, f"-j{os.cpu_count() or 4}"],
                       capture_output=quiet, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle/_ref build failed:\n" + (r.stdout or "") + (r.stderr or ""))
    return available()


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing; run `make -C oracle`")
        L = ctypes.CDLL(LIB_PATH)
        L.solref_last_error.restype = ctypes.c_char_p
        L.solref_load.restype = ctypes.c_void_p
        L.solref_load.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_int]
        L.solref_free.argtypes = [ctypes.c_void_p]
        for f in ("solref_pipeline", "solref_run_reference", "solref_run_compiled", "solref_update_bn_running_stats"):
            getattr(L, f).argtypes = [ctypes.c_void_p]
        L.solref_set_input.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64]
        L.solref_set_param.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64]
        L.solref_numel.restype = ctypes.c_int64
        L.solref_numel.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.solref_get.restype = ctypes.c_int64
        L.solref_get.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64]
        for f in ("solref_graph_json", "solref_partition_json", "solref_param_grads_json"):
            getattr(L, f).argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
        L.solref_oracle_err.restype = ctypes.c_double
        L.solref_oracle_err.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise RefError(lib().solref_last_error().decode())


class RefSession:
    """One reference graph instance (model JSON + SOLW weights at a fixed batch)."""

    def __init__(self, model_json: str, weights: bytes, batch: int, training: bool = False):
        L = lib()
        h = L.solref_load(model_json.encode(), weights, len(weights), batch, int(training))
        if not h:
            raise RefError(L.solref_last_error().decode())
        self.h = h

    def close(self):
        if self.h:
            lib().solref_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def pipeline(self):
        _check(lib().solref_pipeline(self.h))

    def set_input(self, name: str, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.float32)
        _check(lib().solref_set_input(self.h, name.encode(), a.ctypes.data, a.size))

    def set_param(self, name: str, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.float32)
        _check(lib().solref_set_param(self.h, name.encode(), a.ctypes.data, a.size))

    def run_reference(self):
        _check(lib().solref_run_reference(self.h))

    def run_compiled(self):
        _check(lib().solref_run_compiled(self.h))

    def update_bn_running_stats(self):
        _check(lib().solref_update_bn_running_stats(self.h))

    def get(self, name: str, shape=None) -> np.ndarray:
        n = lib().solref_numel(self.h, name.encode())
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, dtype=np.float32)
        got = lib().solref_get(self.h, name.encode(), out.ctypes.data, n)
        if got < 0:
            raise RefError(lib().solref_last_error().decode())
        return out.reshape(shape) if shape is not None else out

    def _json(self, fn) -> object:
        size = 1 << 16
        while True:
            buf = ctypes.create_string_buffer(size)
            rc = fn(self.h, buf, size)
            if rc == 0:
                return json.loads(buf.value.decode())
            if rc < -1:
                size = -rc + 16
                continue
            raise RefError(lib().solref_last_error().decode())

    def graph_json(self):
        return self._json(lib().solref_graph_json)

    def partition(self):
        return self._json(lib().solref_partition_json)

    def param_grads(self):
        return self._json(lib().solref_param_grads_json)


def oracle_err(a: np.ndarray, b: np.ndarray) -> float:
    """The reference's kernel-oracle metric (src/tensor.cpp:324-329), computed by the reference."""
    a = np.ascontiguousarray(a, dtype=np.float32).ravel()
    b = np.ascontiguousarray(b, dtype=np.float32).ravel()
    assert a.size == b.size
    return lib().solref_oracle_err(a.ctypes.data, b.ctypes.data, a.size)
