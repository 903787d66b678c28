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


def test_persist_struct_binding_matches_header():
    """The ctypes mirrors of tps_persist_geom / tps_persist_rank have the C layout."""
    import ctypes
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    lib = nat.load_library()
    assert lib.tps_persist_struct_bytes(0) == ctypes.sizeof(nat.PersistGeom)
    assert lib.tps_persist_struct_bytes(1) == ctypes.sizeof(nat.PersistRank)
    for name, _ in nat.PersistRank._fields_:  # every field the header declares, in order
        assert name in open(HEADER).read()


def test_persist_shape_support_is_host_only():
    """tps_persist_supported / tps_persist_work_bytes need no GPU."""
    import ctypes
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    lib = nat.load_library()
    g = nat.PersistGeom(num_layers=28, hidden=3584, head_dim=128, n_phases=57, rms_eps=1e-6)
    r = nat.PersistRank(nq=4, nkv=1, ffn=2368, vocab=19008, tp=8)
    assert lib.tps_persist_supported(ctypes.byref(g), ctypes.byref(r), 1) == 1
    assert lib.tps_persist_supported(ctypes.byref(g), ctypes.byref(r), 17) == 0   # B > 16
    g64 = nat.PersistGeom(num_layers=2, hidden=256, head_dim=64, n_phases=5, rms_eps=1e-6)
    assert lib.tps_persist_supported(ctypes.byref(g64), ctypes.byref(r), 1) == 0  # head_dim 64
    assert lib.tps_persist_work_bytes(ctypes.byref(g), ctypes.byref(r), 148) > 0
