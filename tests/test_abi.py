"""The C-ABI drop-in boundary (include/solb200.h), checked without a GPU:
 * libsolb200.so loads and exports exactly the entry points the header declares (and the ctypes
   binding names);
 * every struct the header declares has the same size and field offsets in C (compiled here with
   gcc against the header) and in the ctypes mirror;
 * the pure host-side semantics: VirtualPtr offset arithmetic never carries into the reference
   (rt/runtime.cpp:19-24 VirtualPtr::operator+), errors surface through sol_b200_last_error."""
import ctypes as C
import os
import re
import subprocess
import sys

import pytest

from paper_2003_10688_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "solb200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sol_b200_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    return _lib.lib()


def test_header_matches_binding_symbol_list():
    assert _declared() == sorted(_lib.SYMBOLS)


def test_library_exports_every_declared_symbol(L):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(sol_b200_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    for s in _declared():
        assert getattr(L, s) is not None


STRUCTS = {
    "sol_attrs": _lib.Attrs, "sol_unit_op": _lib.UnitOp, "sol_binding": _lib.Binding,
    "sol_unit_desc": _lib.UnitDesc, "sol_module_info": _lib.ModuleInfo,
    "sol_transfer_stats": _lib.TransferStats, "sol_conv_desc": _lib.ConvDesc,
}


def test_struct_layouts_match_header(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void) {']
    for cname, py in STRUCTS.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", str(src), "-o", str(exe)], check=True)
    want = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = line.split()
        want[(s, f)] = int(v)
    for cname, py in STRUCTS.items():
        assert C.sizeof(py) == want[(cname, "size")], cname
        for f, _ in py._fields_:
            assert getattr(py, f).offset == want[(cname, f)], (cname, f)


def test_vptr_add_semantics(L):
    out = C.c_uint64()
    ref = 7 << 32
    assert L.sol_b200_vptr_add(ref | 100, 28, C.byref(out)) == _lib.SOL_OK
    assert out.value == ref | 128
    assert L.sol_b200_vptr_add(ref | 0xFFFFFFF0, 0xF, C.byref(out)) == _lib.SOL_OK
    assert out.value == ref | 0xFFFFFFFF
    # an offset that would carry into the reference id is an overflow, not a different buffer
    assert L.sol_b200_vptr_add(ref | 0xFFFFFFF0, 0x10, C.byref(out)) == _lib.SOL_E_OVERFLOW
    assert b"overflow" in L.sol_b200_last_error()
    assert L.sol_b200_vptr_add(ref, 1 << 32, C.byref(out)) == _lib.SOL_E_OVERFLOW


def test_status_codes_match_header():
    text = open(HEADER).read()
    for name in ("SOL_OK", "SOL_E_USE_AFTER_FREE", "SOL_E_UNKNOWN_REF", "SOL_E_OUT_OF_BOUNDS",
                 "SOL_E_INVALID_ARGUMENT", "SOL_E_SHAPE_MISMATCH", "SOL_E_UNSUPPORTED", "SOL_E_OVERFLOW",
                 "SOL_E_OUT_OF_REFS", "SOL_E_NCCL", "SOL_E_CUDA"):
        m = re.search(rf"\b{name}\s*=\s*(\d+)", text)
        assert m, name
        assert int(m.group(1)) == getattr(_lib, name), name


def test_product_path_fails_loudly_without_library(tmp_path):
    """No CPU fallback: importing the binding against a missing library raises."""
    code = ("import paper_2003_10688_b200._lib as l; l.LIB_PATH = '/nonexistent/libsolb200.so'\n"
            "try:\n    l.lib()\nexcept FileNotFoundError:\n    print('raised')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert "raised" in r.stdout, r.stderr
