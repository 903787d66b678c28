"""CPU checks of the C-ABI boundary: the library loads and exports every symbol the header declares."""

import os
import re
import subprocess

import pytest

from paper_2605_23945_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tpshift_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tps_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(nat.SIGNATURES), "ctypes signatures must mirror include/tpshift_b200.h"


def test_library_exports_every_declared_symbol():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built (run make / __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tps_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    lib = nat.load_library()
    assert b"sm_100a" in lib.tps_version()
    # host-only helpers work without a GPU
    assert lib.tps_linear_splits(4608, 3584, 64) >= 1
    assert lib.tps_attn_splits(1, 4, 136) == -1       # tail: one CTA cluster per (row, kv head)
    assert lib.tps_attn_splits(96, 4, 136) == 0       # page-balanced schedule
    assert lib.tps_attn_splits(300, 1, 136) == 0      # more segments than CTA slots: page-balanced
    assert 1 <= lib.tps_attn_splits(4, 4, 136) <= 32  # fixed split-KV


def test_status_codes_map_to_tpshift_errors():
    from paper_2605_23945_b200.errors import ConfigError, PlanVerificationError
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    nat.load_library()
    with pytest.raises(ConfigError):
        nat.check(nat.TPS_EINVAL, "x")
    with pytest.raises(PlanVerificationError):
        nat.check(nat.TPS_EPLAN, "x")
    with pytest.raises(RuntimeError):
        nat.check(nat.TPS_ECUDA, "x")


def test_sm100a_code_in_library():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "-sass", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out      # tcgen05.mma (5th-gen tensor cores)
    assert "UTMALDG" in out      # TMA tensor loads
    assert "LDTM" in out         # tcgen05.ld (TMEM -> registers)
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", nat.LIB_PATH], capture_output=True,
                                       text=True).stdout
