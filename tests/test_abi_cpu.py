"""The C-ABI library loads without a GPU and exports every symbol
``include/mosel_b200.h`` declares; no compute calls are made here."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "mosel_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ms_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_18481_b200 import build, device
    build.build()
    return device.lib()


def test_header_declares_the_entry_points():
    names = _declared()
    for must in ("ms_policy_select", "ms_compact", "ms_compact_index", "ms_gather_rows",
                 "ms_gemm_plan_dense", "ms_gemm_plan_conv", "ms_gemm_plan_gather", "ms_gemm_run",
                 "ms_program_run", "ms_event_record", "ms_event_elapsed_us"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing


def test_python_binding_covers_the_header(lib):
    from paper_2310_18481_b200 import device
    assert set(_declared()) <= set(device.EXPORTS)


def test_abi_version_and_error_plumbing(lib):
    from paper_2310_18481_b200 import device
    assert lib.ms_abi_version() == 4
    # invalid arguments are rejected before any CUDA call, with a message
    rc = lib.ms_policy_select(None, None, None, 0, None, 0, 1.0, 4, None, None)
    assert rc == 1
    assert b"bad shape" in lib.ms_last_error()
    with pytest.raises(device.DeviceError, match="bad shape"):
        device.check(rc, "ms_policy_select")
    rc = lib.ms_compact_index(None, 4, 9, None, None, None, None, None, None)
    assert rc == 1 and b"K must be" in lib.ms_last_error()


def test_op_records_build_without_a_device(lib):
    from paper_2310_18481_b200 import device
    buf = ctypes.create_string_buffer(device.OP_BYTES + 64)
    addr = (ctypes.addressof(buf) + 63) & ~63
    assert lib.ms_op_pool2d(addr, None, 1, 8, 8, 64, 64, 3, 2, 0, 1, 1, None, 64, 0) == 0
    assert lib.ms_op_segment_mean(addr, None, 1, 3, 49, 64, None, 64) == 0
    assert lib.ms_op_im2col(addr, None, 1, 8, 8, 3, 7, 7, 2, 3, None, 192) == 0


def test_no_cpu_fallback_without_cuda(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2310_18481_b200 import device
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        device.policy_select([[1]], None, [1], [10], 0, 1.0)
