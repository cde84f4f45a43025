"""The C-ABI library loads on a CPU-only host and exports every function
include/nvrec_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from helpers import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "nvrec_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(nvrec_\w+)\s*\(",
                                 src, re.M)))


def test_header_declares_the_abi():
    names = _declared()
    assert {"nvrec_model_create", "nvrec_model_load", "nvrec_forward_f32",
            "nvrec_recover_u8", "nvrec_loss_mask", "nvrec_workspace_bytes",
            "nvrec_last_error", "nvrec_abi_version", "nvrec_model_destroy"} <= set(names)


def test_library_exports_every_declared_symbol():
    from paper_2604_27441_b200 import _native
    lib = _native.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_native.EXPORTS) == set(_declared())
    assert lib.nvrec_abi_version() == _native.ABI_VERSION == 5


def test_sm100a_code_only():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2604_27441_b200 import _native
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
