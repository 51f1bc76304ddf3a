"""The interface generators (paper_1810_09891_b200/abi.py) against the
reference's own ABI description (tests/golden/abi_reference.json, from
nfftk.abi.interface_json()) and against the ctypes table of _lib.py."""

import ctypes
import json
import os
import subprocess

import pytest

from conftest import GOLDEN
from paper_1810_09891_b200 import _lib, abi

REF = json.load(open(os.path.join(GOLDEN, "abi_reference.json")))

CTYPE = {"int32_t": ctypes.c_int32, "int64_t": ctypes.c_int64, "uint32_t": ctypes.c_uint32,
         "uint64_t": ctypes.c_uint64, "double": ctypes.c_double}


def test_reference_symbols_identical():
    ours = {f["name"]: f for f in json.loads(abi.interface_json())["functions"]}
    assert [f["name"] for f in REF["functions"]] == abi.REFERENCE_SYMBOLS
    for f in REF["functions"]:
        o = ours[f["name"]]
        assert o["returns"].replace(" ", "") == f["returns"].replace(" ", "")
        assert [(a["type"].replace(" ", ""), a["name"]) for a in o["args"]] == \
               [(a["type"].replace(" ", ""), a["name"]) for a in f["args"]]
        assert not o["extension"]
    assert json.loads(abi.interface_json())["error_codes"] == REF["error_codes"]
    assert abi.abi_version() == REF["abi_version"]


def test_header_declarations_match_ctypes_table():
    fs = abi.functions()
    assert [f[0] for f in fs] == list(_lib.SIGNATURES)
    for name, ret, args, doc in fs:
        restype, argtypes = _lib.SIGNATURES[name]
        assert len(args) == len(argtypes), name
        for (t, _), ct in zip(args, argtypes):
            if "*" in t:  # pointers: any ctypes pointer flavour
                assert ct in (ctypes.c_void_p, ctypes.c_char_p) or hasattr(ct, "_type_"), (name, t)
            else:
                assert ct is CTYPE[t], (name, t, ct)
        assert doc, f"{name} has no doc comment"


def test_generated_header_compiles_and_json_is_complete(tmp_path):
    h = tmp_path / "nfftk_flat.h"
    j = tmp_path / "nfftk.json"
    assert abi.main(["--emit-header", str(h), "--emit-json", str(j)]) == 0
    r = subprocess.run(["gcc", "-fsyntax-only", "-x", "c", str(h)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    doc = json.loads(j.read_text())
    assert len(doc["functions"]) == len(_lib.SIGNATURES)
    assert sum(not f["extension"] for f in doc["functions"]) == 13
    with pytest.raises(SystemExit):
        abi.main([])
