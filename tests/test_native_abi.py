"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/ott_b200.h declares; host-side config/error behaviour mirrors the
reference (no GPU compute here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_symbols():
    src = "".join(open(os.path.join(ROOT, "include", f)).read() for f in ("ott_b200.h", "ott_model.h"))
    return sorted(set(re.findall(r"\b(ott_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2505_10938_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_native.EXPORTED) == set(syms)


def test_record_bytes_and_version_without_gpu():
    from paper_2505_10938_b200 import _native

    L = _native.lib()
    assert L.ott_record_bytes(128, 32, 2) == 32 * 128 // 2 + 8 * 128 + 8 * 32
    assert L.ott_record_bytes(64, 128, 2) == 128 * 64 // 2 + 8 * 64 + 8 * 128
    assert b"sm_100a" in L.ott_version()
    assert L.ott_cache_struct_bytes() == ctypes.sizeof(_native.OttCacheT)


def test_contract_errors_map_to_contract_violation():
    from paper_2505_10938_b200 import ContractViolation, _native

    c = _native.OttCacheT(n_units=1, head_dim=128, group_size=32, residual=0, capacity=0, aux_capacity=0, bits=9)
    with pytest.raises(ContractViolation):  # bits outside [1, 8] (quant.py:53-54)
        _native.check(_native.lib().ott_flush(ctypes.byref(c), 0, 1, 0, None, None, 0, 0, None))
    c.bits = 2
    with pytest.raises(ContractViolation):  # null state buffers
        _native.check(_native.lib().ott_flush(ctypes.byref(c), 0, 1, 0, None, None, 0, 0, None))


def test_engine_config_mirrors_reference():
    from paper_2505_10938_b200 import ContractViolation, EngineConfig

    cfg = EngineConfig()
    assert (cfg.bits, cfg.group_size, cfg.residual, cfg.outlier_num, cfg.aux_capacity) == (2, 128, 32, 3, 32)
    assert cfg.skip_layers == (0, 1) and cfg.outlier_capacity(0) == 0 and cfg.outlier_capacity(2) == 3
    for bad in (dict(bits=0), dict(group_size=0), dict(residual=-1), dict(head_dim=0)):
        with pytest.raises(ContractViolation):
            EngineConfig(**bad)
    assert issubclass(ContractViolation, ValueError)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2505_10938_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
                assert "ott_oracle" not in src, f


def test_split_policy_without_gpu():
    """ott_pick_splits is host arithmetic (148 SMs assumed without a device): the split counts the
    measured sweeps chose (profiles/r2_shard_splits.log, r2_pick_splits.log) for the BASELINE
    shapes. 1,024 units run the tail schedule with thirds; 256-592 units at long contexts aim at
    ~1,024 quantized CTAs; short contexts keep ~3 CTAs per SM."""
    from paper_2505_10938_b200 import _native

    L = _native.lib()

    def pick(units, tokens, bits=2, d=128, G=32):
        c = _native.OttCacheT(n_units=units, head_dim=d, group_size=G, residual=128, capacity=32, aux_capacity=32,
                              bits=bits)
        return L.ott_pick_splits(ctypes.byref(c), 8, tokens)

    assert pick(1024, 16384) == 3  # config 4 at N = 1: tail schedule
    assert pick(512, 16384) == 2   # config-4 shard at N = 2
    assert pick(256, 16384) == 4   # N = 4
    assert pick(128, 16384) == 3   # N = 8
    assert pick(128, 4096) == 3 and pick(512, 8192) == 1  # config 3
    assert pick(256, 2304) == 2    # config 1 layer (B = 8, H = 32)
    assert pick(32, 1024) == 1     # config 0
    assert pick(1024, 16384, bits=4) == 1  # the tail schedule is the 2-bit kernel's
