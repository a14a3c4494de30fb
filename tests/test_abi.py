"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/bpx.h declares (no compute calls: this runs without a GPU)."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bpx.h")
LIB = os.path.join(ROOT, "paper_2112_10065_b200", "libbpx.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"BPX_API\s+[\w\s\*]*?\b(bpx_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2112_10065_b200 import build
    build.build()
    from paper_2112_10065_b200 import ops
    return ops.load_library()


def test_header_declares_the_surface():
    names = declared()
    for must in ("bpx_conv3x3_fwd", "bpx_conv3x3_dgrad", "bpx_conv3x3_wgrad",
                 "bpx_linear_fwd", "bpx_linear_dgrad", "bpx_linear_wgrad",
                 "bpx_maxpool2x2_fwd", "bpx_maxpool2x2_bwd", "bpx_maxpool2x2_fwd_idx",
                 "bpx_maxpool2x2_bwd_idx", "bpx_softmax_xent",
                 "bpx_sgd_update", "bpx_reshard_pull", "bpx_allreduce_sum_prefix",
                 "bpx_signal_barrier", "bpx_status_string"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB]).decode()
    exported = set(re.findall(r"\sT\s(bpx_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert getattr(lib, n) is not None


def test_ctypes_table_matches_header(lib):
    from paper_2112_10065_b200 import ops
    assert sorted(ops.EXPORTED) == declared()


def test_status_strings_and_version(lib):
    assert lib.bpx_abi_version() == 1
    assert lib.bpx_status_string(0) == b"BPX_OK"
    assert lib.bpx_status_string(4) == b"BPX_ERR_WORKSPACE"
    assert lib.bpx_status_string(99) == b"BPX_ERR_UNKNOWN"


def test_built_for_sm100a_only():
    out = subprocess.check_output(["cuobjdump", "--list-elf", LIB]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_argument_validation_without_gpu(lib):
    # invalid arguments are rejected before any CUDA call
    assert lib.bpx_conv3x3_fwd(None, None, None, None, 1, 8, 8, 8, 8, 1, None, 0,
                               None) == 1
    assert lib.bpx_reshard_pull(None, None, None, None, None, 65, None) == 1


@pytest.mark.parametrize("n,h,cin,cout", [(2, 17, 32, 32), (2, 8, 32, 32), (1, 5, 4, 4),
                                          (2, 35, 128, 32), (2, 9, 16, 16), (3, 7, 3, 64),
                                          (2, 224, 64, 64), (0, 4, 8, 8)])
def test_workspace_queries_any_shape(lib, n, h, cin, cout):
    """Workspace queries are host-only and must answer for every shape the
    dispatch may see (the first engine's planner may not apply to it)."""
    for f in ("bpx_conv3x3_fwd_workspace", "bpx_conv3x3_dgrad_workspace",
              "bpx_conv3x3_wgrad_workspace"):
        assert getattr(lib, f)(n, h, h, cin, cout) >= 0
    for f in ("bpx_linear_fwd_workspace", "bpx_linear_dgrad_workspace",
              "bpx_linear_wgrad_workspace"):
        assert getattr(lib, f)(n * h * h, cin, cout) >= 0
