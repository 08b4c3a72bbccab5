"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, and exports exactly the
symbols include/tl_api.h declares; error paths return status codes instead of crashing."""
import ctypes as C
import os
import re

import pytest

from paper_2503_20313_b200 import _lib
from paper_2503_20313_b200 import build as B

HEADER = os.path.join(B.ROOT, "include", "tl_api.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tl_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("tl_ag_gemm", "tl_gemm_rs", "tl_mlp_forward", "tl_comm_create", "tl_comm_connect",
              "tl_comm_destroy", "tl_comm_check", "tl_set_option"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for f in header_functions():
        assert hasattr(L, f), f"{f} declared in tl_api.h but not exported"
    # and the binding declares a signature for each of them
    assert set(header_functions()) == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", B.LIB], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "UBLKCP"):
        assert mnemonic in sass, f"{mnemonic} missing: not a tcgen05/TMA build"


def test_status_strings_and_handle():
    L = _lib.lib()
    names = [L.tl_status_string(i).decode() for i in range(6)]
    assert names == _lib.STATUS_NAMES
    assert L.tl_handle_size() >= 64 + 8
    assert b"sm_100a" in L.tl_build_info()


def test_errors_without_device_are_codes_not_crashes():
    L = _lib.lib()
    h = C.c_void_p()
    buf = C.create_string_buffer(L.tl_handle_size())
    # invalid arguments are rejected before touching CUDA
    assert L.tl_comm_create(3, 2, 0, 256, 128, buf, C.byref(h)) == _lib.TL_ERR_INVALID
    assert L.tl_comm_create_loopback(2, 0, 256, 128, None) == _lib.TL_ERR_INVALID
    assert L.tl_comm_create_loopback(9, 0, 256, 128, C.byref(h)) in (_lib.TL_ERR_UNSUPPORTED, _lib.TL_ERR_CUDA)
    assert L.tl_ag_gemm(None, None, None, None, None, 8, 8, 8, None) == _lib.TL_ERR_INVALID
    assert L.tl_set_option(None, b"cta_pair", 2) == _lib.TL_ERR_INVALID
    assert L.tl_comm_destroy(None) == _lib.TL_OK


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU box: covered by -m gpu")
def test_no_device_reports_cuda_error():
    L = _lib.lib()
    h = C.c_void_p()
    st = L.tl_comm_create_loopback(2, 0, 256, 128, C.byref(h))
    assert st == _lib.TL_ERR_CUDA
    assert L.tl_last_error()


def test_binding_rejects_host_and_mistyped_tensors_before_the_abi():
    """The C ABI takes untyped pointers; the binding must refuse host memory, wrong dtypes,
    non-contiguous views and inconsistent shapes before any pointer crosses it."""
    import torch
    import paper_2503_20313_b200 as tl
    from paper_2503_20313_b200 import _check_mlp, _check_rs, _dev
    x = torch.zeros(64, 128, dtype=torch.bfloat16)                         # host tensor
    with pytest.raises(ValueError, match="CUDA"):
        _check_mlp(2, 0, x, x, x, x, None, tl.ACT_SILU_MUL)
    with pytest.raises(ValueError, match="CUDA"):
        _check_rs(1, 0, torch.zeros(8, 8, dtype=torch.float32), x, x)
    with pytest.raises(TypeError):
        _dev([1, 2], "A", torch.bfloat16, (None,))
