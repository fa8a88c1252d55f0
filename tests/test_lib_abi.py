"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/kvc.h declares, and the ctypes structures match the C layout."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvc.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(kvc_\w+)\(", text, re.M)))


def test_header_matches_binding_table():
    from paper_2410_00161_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    from paper_2410_00161_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libkvc.so not built (run __graft_entry__.build())")
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.kvc_abi_version() == 3
    assert lib.kvc_status_name(1).decode() == "PreemptionNeeded"


def test_ctypes_layout_matches_c():
    from paper_2410_00161_b200 import _lib

    structs = {"kvc_pool": _lib.KvcPool, "kvc_decode_args": _lib.DecodeArgs,
               "kvc_window_args": _lib.WindowArgs, "kvc_evict_args": _lib.EvictArgs,
               "kvc_full_args": _lib.FullArgs, "kvc_dense_args": _lib.DenseArgs,
               "kvc_attn_metric_args": _lib.AttnMetricArgs}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "l.c")
        exe = os.path.join(tmp, "l")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-o", exe, src], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split("\n")
    got = dict(line.split() for line in out if line)
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)
