"""CPU-side checks of the boundary: libensi.so builds, loads, and exports every symbol include/ensi.h declares;
the product package never touches oracle/.  No compute calls (there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ensi.h")
PKG = os.path.join(ROOT, "paper_2509_09424_b200")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^ENSI_API\s+[\w\s\*]+?\b(ensi_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2509_09424_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    names = _declared()
    for required in ["ensi_ctx_create", "ensi_load_keys", "ensi_pcmm_ternary", "ensi_decrypt_debug"]:
        assert required in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath]).decode()
    exported = set(re.findall(r" T (ensi_\w+)", out))
    assert set(_declared()) == exported      # nothing undeclared leaks out of the ABI


def test_binding_lists_every_symbol(libpath):
    from paper_2509_09424_b200 import ensi
    assert sorted(ensi.EXPORTS) == _declared()
    assert ensi.lib().ensi_abi_version() == 2


def test_sm100a_code_in_library(libpath):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath]).decode()
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
                assert "liboracle" not in txt, f
                assert "ensi_oracle" not in txt, f
