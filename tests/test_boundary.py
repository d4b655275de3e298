"""CPU-side checks of the C-ABI boundary (no GPU, no compute calls).

libcsk.so builds for sm_100a, loads, and exports every function include/csk.h
declares; the product package never reaches into oracle/ (the oracle is test
infrastructure) and has no CPU fallback.
"""
import ctypes
import os
import re
import subprocess

import paper_2508_14209_b200.csk as csk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2508_14209_b200")


def test_library_exports_every_header_symbol():
    L = csk.lib()
    syms = csk.header_symbols()
    assert {"cs_plan", "cs_apply", "ms_apply", "ms_solve", "ms_lstsq", "ne_lstsq"} <= set(syms)
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_status_strings_and_version():
    L = csk.lib()
    for code, name in csk._STATUS_NAMES.items():
        assert L.csk_status_str(code).decode() == name
    assert b"sm_100a" in L.csk_version()


def test_null_plan_rejected_without_gpu():
    # argument validation happens before any CUDA call
    L = csk.lib()
    assert L.cs_plan_info(None, None, None, None) == csk.EINVAL
    assert b"plan is NULL" in L.csk_last_error()
    assert L.cs_apply(None, 0, 1, None, 1, None, None, 1, -1, None) == csk.EINVAL


def test_sass_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", csk._build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_product_never_uses_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), f
                assert "liboracle" not in text, f
                assert "oracle.c" not in text, f


def test_binding_has_no_cpu_fallback():
    text = open(os.path.join(PKG, "csk.py")).read()
    assert "no CPU fallback" in text
    assert "numpy.linalg" not in text and "np.linalg" not in text


def test_binding_arity_matches_header():
    # every function the binding declares argtypes for takes exactly as many parameters as csk.h says
    hdr = open(os.path.join(ROOT, "include", "csk.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    decls = {}
    for m in re.finditer(r"\b(?:csk_status|void|const char\*|uint64_t)\s+(\w+)\s*\(([^;{]*?)\)\s*;", hdr):
        params = [p for p in m.group(2).split(",") if p.strip() and p.strip() != "void"]
        decls[m.group(1)] = len(params)
    L = csk.lib()
    checked = 0
    for name, n in decls.items():
        f = getattr(L, name, None)
        if f is not None and getattr(f, "argtypes", None) is not None:
            assert len(f.argtypes) == n, (name, len(f.argtypes), n)
            checked += 1
    assert checked >= 20, checked


def test_binding_constants_match_header():
    # status codes, variants and plan flags the binding passes across the ABI equal csk.h's
    hdr = open(os.path.join(ROOT, "include", "csk.h")).read()
    flags = {m.group(1): int(m.group(2), 16) for m in re.finditer(r"#define CSK_PLAN_(\w+)\s+0x([0-9a-fA-F]+)u", hdr)}
    assert flags.get("SORT") == csk.PLAN_SORT and flags.get("HASH") == csk.PLAN_HASH, flags
    body = hdr[hdr.index("typedef enum {"):hdr.index("} csk_status;")]
    status = {m.group(1): int(m.group(2)) for m in re.finditer(r"CSK_(\w+)\s*=\s*(\d+)", body)}
    for name in ("OK", "EINVAL", "ESHAPE", "EDTYPE", "ENOMEM", "ECUDA", "ENOTPD", "ESINGULAR", "EUNSUPPORTED"):
        assert status[name] == getattr(csk, name), name
