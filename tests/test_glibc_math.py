"""The transport's log / sin / cos restated from the host libm
(csrc/glibc_math.cuh): the host build of the same header against libm itself,
bit for bit, on 2e6 transport arguments per function (log on (0, 1] and its
near-1 branch, sin/cos on (0, 2 pi]) and around every branch threshold.  The
device build is checked against libm in tests/test_gpu_api.py and through
whole transport histories in tests/test_transport_gpu.py."""

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2504_19048_b200" / "csrc"


def test_tables_come_from_this_libm():
    from paper_2504_19048_b200 import glibc_tables
    t = glibc_tables.read_tables()
    if t is None:
        pytest.skip("host libm is not the glibc build the restatement was taken from")
    log_tab, sc = t
    assert len(log_tab) == 256 and len(sc) == 440


def test_host_restatement_equals_libm(tmp_path):
    from paper_2504_19048_b200 import glibc_tables
    inc = tmp_path / "glibc_tables.inc"
    if not glibc_tables.generate(inc):
        pytest.skip("host libm is not the glibc build the restatement was taken from")
    # the header's own directory must not shadow the temporary tables
    hdr = tmp_path / "glibc_math.cuh"
    hdr.write_text((CSRC / "glibc_math.cuh").read_text())
    exe = tmp_path / "selftest"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-builtin",
                    "-I", str(tmp_path), str(ROOT / "tests" / "native" / "glibc_math_selftest.cpp"),
                    "-o", str(exe), "-ldl", "-lm"], check=True)
    r = subprocess.run([str(exe), "2000000", "20261017"], capture_output=True, text=True)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    for fn in ("log", "sin", "cos"):
        assert f"{fn} checked" in r.stdout and "mismatches 0" in r.stdout
