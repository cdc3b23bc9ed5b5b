"""The C-ABI library loads without a GPU and exports every symbol that
include/ttb.h declares; host-only entry points behave."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2507_14668_b200 import _native as nat
from paper_2507_14668_b200.build import build

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    build()
    return nat.load()


def header_functions():
    text = (ROOT / "include" / "ttb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ttb_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported(lib):
    declared = header_functions()
    assert len(declared) >= 15
    assert sorted(nat.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ttb_\w+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing


def test_sm100a_code_present(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points(lib):
    assert lib.ttb_abi_version() == 1
    assert lib.ttb_strerror(-2) == b"index outside [0, rows)"
    g = nat.TtbGeom()
    for k, (m, n) in enumerate(zip((200, 200, 250), (4, 4, 4))):
        g.m[k], g.n[k] = m, n
    for k, r in enumerate((1, 32, 32, 1)):
        g.r[k] = r
    nbytes = C.c_size_t()
    assert lib.ttb_workspace_bytes(C.byref(g), 65536, 65536, C.byref(nbytes)) == 0
    assert 50e6 < nbytes.value < 1e9
    g.r[0] = 2  # boundary rank must be 1
    assert lib.ttb_workspace_bytes(C.byref(g), 65536, 65536, C.byref(nbytes)) == nat.TTB_EINVAL
    g.r[0] = 1
    g.m[0] = 1 << 20  # rows >= 2^31 rejected
    assert lib.ttb_workspace_bytes(C.byref(g), 65536, 65536, C.byref(nbytes)) == nat.TTB_EINVAL
    # NULL handles are rejected, not dereferenced
    assert lib.ttb_plan(None, None, 1, None, 1, 1, None) == nat.TTB_EINVAL
    assert lib.ttb_forward(None, None, None, None, None, None) == nat.TTB_EINVAL


def test_check_maps_to_reference_exceptions():
    with pytest.raises(ValueError):
        nat.check(nat.TTB_ERANGE)
    with pytest.raises(ValueError):
        nat.check(nat.TTB_EEMPTY)
    with pytest.raises(RuntimeError):
        nat.check(nat.TTB_ECUDA)
    assert isinstance(nat.errbits_to_exception(nat.ERRBIT_EMPTY_BAG), ValueError)
