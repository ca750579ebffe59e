"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every symbol include/b200tally.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2504_19048_b200 import _lib, build

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "b200tally.h").read_text()
    return sorted(set(re.findall(r"^(?:bt_status|const char \*)\s*(bt_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == header_symbols()


def test_library_exports_every_header_symbol():
    build.build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in _lib.load().bt_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_19048_b200 import MeshTally, build_cube_mesh
    with pytest.raises((RuntimeError, ValueError)):
        MeshTally(build_cube_mesh(2), 10)
