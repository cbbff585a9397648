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
    assert ensi.lib().ensi_abi_version() == 5


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


def test_wire_host_serialisation_round_trip():
    """The wire format keeps the low ceil(bits/8) bytes of each canonical word, limb blocks in order (numpy, CPU)."""
    import numpy as np
    from paper_2509_09424_b200.ensi import wire_pack_host, wire_unpack_host
    rs = np.random.default_rng(3)
    widths = [7, 5, 5, 6]
    n, level = 32, 4
    x = np.stack([rs.integers(0, 1 << (8 * w - 1), (2, 2, n), dtype=np.uint64) for w in widths], axis=2)
    p = wire_pack_host(x, widths)
    assert p.shape == (2, 2 * n * sum(widths))
    # limb 1 of poly 0 of ciphertext 0 starts after limb 0's n * 7 bytes; word 3 is little-endian
    off = n * widths[0] + 3 * widths[1]
    assert int.from_bytes(p[0, off:off + widths[1]].tobytes(), "little") == int(x[0, 0, 1, 3])
    assert (wire_unpack_host(p, widths, level, n) == x).all()
