"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol include/sparsekit_b200.h declares (no compute calls without a GPU)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "sparsekit_b200.h")
LIB = os.path.join(ROOT, "paper_2509_20883_b200", "libsparsekit_b200.so")


def header_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^(?:int|uint64_t|int64_t|const char\*)\s+(skb_\w+)\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-j8"], cwd=os.path.join(ROOT, "paper_2509_20883_b200", "csrc"), check=True)
    from paper_2509_20883_b200 import _native
    return _native.load_library()


def test_header_declares_symbols():
    syms = header_symbols()
    assert len(syms) >= 40
    assert "skb_table_lookup_or_insert" in syms and "skb_fused_forward" in syms


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (skb_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_python_binding_covers_header(lib):
    from paper_2509_20883_b200 import _native
    assert sorted(_native.EXPORTED) == header_symbols()
    for s in header_symbols():
        assert getattr(lib, s) is not None


def test_host_only_entry_points(lib):
    # pure host helpers callable without a device
    assert lib.skb_version().decode().startswith("sparsekit_b200")
    assert lib.skb_fnv1a64_host(b"a", 1) == 0xAF63DC4C8601EC8C
    assert lib.skb_fnv1a64_host(b"", 0) == 0xCBF29CE484222325


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2509_20883_b200 as skb
    with pytest.raises(RuntimeError, match="CUDA"):
        skb.EmbeddingTable("t", 4)
