"""Host-side checks of the C ABI (-m "not gpu"): the in-tree library builds,
loads and exports every symbol include/vsaogm.h declares; host argument
validation works without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2408_09066_b200 import _build
    _build.build()
    from paper_2408_09066_b200 import vsaogm
    return vsaogm.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "vsaogm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vsaogm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("vsaogm_create", "vsaogm_encode_bundle", "vsaogm_decode", "vsaogm_entropy"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    from paper_2408_09066_b200.vsaogm import EXPORTS
    syms = header_symbols()
    assert sorted(EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only(lib):
    import subprocess
    from paper_2408_09066_b200.vsaogm import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_strerror_and_host_validation(lib):
    from paper_2408_09066_b200.vsaogm import Bounds, EINVAL_ARG, EINVAL_DIM, strerror
    assert strerror(0) == "ok"
    assert "dimension" in strerror(EINVAL_DIM)
    ctx = ctypes.c_void_p()
    b = Bounds(0.0, 0.0, 10.0, 10.0)
    assert lib.vsaogm_create(0, 0, 0.2, b, ctypes.byref(ctx)) == EINVAL_DIM
    assert lib.vsaogm_create(16, 0, 0.0, b, ctypes.byref(ctx)) == EINVAL_ARG
    assert lib.vsaogm_create(16, 0, -1.0, b, ctypes.byref(ctx)) == EINVAL_ARG
    assert lib.vsaogm_create(16, 0, 0.2, Bounds(0.0, 0.0, 0.0, 10.0), ctypes.byref(ctx)) == EINVAL_ARG
    assert lib.vsaogm_create(16, 0, 0.2, Bounds(0.0, 0.0, float("nan"), 10.0), ctypes.byref(ctx)) == EINVAL_ARG
    assert lib.vsaogm_encode_bundle(None, None, None, 5) == EINVAL_ARG
    assert lib.vsaogm_test_gemm(None, None, 1, 1, 64, 0, -1, 0, 0, None, None) == EINVAL_ARG
    assert lib.vsaogm_set_tuning(None, b"gemm_bn", 0) == EINVAL_ARG


def test_oracle_and_product_share_no_code():
    # the oracle is plain C with its own RNG; the CUDA sources never include it and vice versa
    csrc = os.path.join(ROOT, "paper_2408_09066_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        assert "oracle" not in txt.lower().replace("the oracle never", "")
    orc = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "#include \"" not in orc
    for f in ("vsaogm.py", "parallel.py", "__init__.py"):
        txt = open(os.path.join(ROOT, "paper_2408_09066_b200", f)).read()
        assert "import oracle" not in txt and "from oracle" not in txt
