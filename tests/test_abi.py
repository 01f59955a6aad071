"""CPU checks of the boundary: the C-ABI libraries load and export every
function include/h2d.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

import helpers

HEADER = os.path.join(helpers.ROOT, "include", "h2d.h")
# product-only: benchmark support, the block decomposition, and the field / checkpoint I/O
# (the I/O is checked against the reference writer itself, tests/test_io.py)
PRODUCT_ONLY_PREFIXES = ("launch_count", "step_timed", "flush_l2", "create_block", "block_", "halo_",
                         "write_fields", "diag_line", "save_state", "load_state", "comm_", "blocks_run",
                         "nccl_unique_id")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(?:int|void|long long)\s+h2d_(\w+)\s*\(", text)))


def test_header_declares_reference_entry_points():
    names = declared()
    for must in ("create", "destroy", "upload_state", "download_state", "fill_ghosts", "sync_derived",
                 "update_interface_normals", "cfl_dt", "lagrange_step", "set_lagrange", "remap_step", "run",
                 "totals", "last_error"):
        assert must in names


def test_product_library_exports_every_symbol():
    if not os.path.exists(helpers.PRODUCT_LIB):
        from paper_2208_13409_b200 import build
        build.build()
    dll = ctypes.CDLL(helpers.PRODUCT_LIB)
    missing = [n for n in declared() if not hasattr(dll, "h2d_" + n)]
    assert missing == []
    assert dll.h2d_abi_version() == 3


# the reference's sub-step entry points and scalar kernels: checked against the
# reference library itself (h2dr_, tests/test_substeps.py), not the restatement
PRODUCT_AND_REF = ("predict", "correct", "remap_single_axis", "scalar_eval")


def test_oracle_library_exports_the_same_abi(orc):
    missing = [n for n in declared() if not n.startswith(PRODUCT_ONLY_PREFIXES) and n not in PRODUCT_AND_REF
               and not hasattr(orc.dll, "h2do_" + n)]
    assert missing == []


def test_reference_shim_exports_the_substep_entry_points(ref):
    missing = [n for n in PRODUCT_AND_REF if not hasattr(ref.dll, "h2dr_" + n)]
    assert missing == []


def test_product_fails_loudly_without_a_device():
    """No CPU fallback: creating a context with no CUDA device is an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2208_13409_b200 import abi, errors, make_config
    lib = abi.Library(helpers.PRODUCT_LIB, "h2d_")
    with pytest.raises(errors.DeviceError):
        abi.Solver(lib, make_config(8, 8, 1.0, 1.0))
