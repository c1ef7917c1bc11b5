"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/il.h declares
(no compute calls: runs without a GPU)."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "il.h")).read()
    return sorted(set(re.findall(r"^(?:il_status|const char\*)\s+(il_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ["il_pool_load", "il_refine_batch", "il_prefix_match", "il_prefill_attn", "il_commit"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2507_08523_b200 import build, _lib
    lib = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = set(re.findall(r"\bT (il_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(declared())
    L = _lib.load()                                    # dlopen works without a GPU
    for n in declared():
        assert hasattr(L, n)


def test_sass_is_sm100a():
    from paper_2507_08523_b200 import build
    lib = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib]).decode()
    assert "sm_100a" in out


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2507_08523_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle/" not in txt and "liboracle" not in txt, f
