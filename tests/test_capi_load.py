"""The C-ABI library loads and exports every symbol include/moqe_gpu.h declares.
No compute calls (CPU container has no GPU); pure host helpers only."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moqe_gpu.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moqe_gpu_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_02410_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2310_02410_b200.build import build
        build()
    return _lib.load()


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("moqe_gpu_quantize_pack", "moqe_gpu_pack", "moqe_gpu_unpack", "moqe_gpu_route",
              "moqe_gpu_bank_create", "moqe_gpu_moe_forward", "moqe_gpu_moe_forward_host"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_binding_table_matches_header():
    from paper_2310_02410_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_host_helpers_without_gpu(lib):
    assert lib.moqe_gpu_abi_version() == 1
    # bitpack.cpp:12-16 sizes
    assert [lib.moqe_gpu_packed_size(b, n) for b, n in ((2, 0), (8, 5), (4, 5), (2, 5), (3, 8), (3, 9), (3, 5))] == \
        [0, 5, 3, 2, 3, 6, 3]
    assert lib.moqe_gpu_packed_size(5, 1) == ctypes.c_size_t(-1).value
    assert lib.moqe_gpu_status_string(1) == b"invalid_argument"


def test_library_is_sm100a():
    from paper_2310_02410_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
