"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/sqf2k_b200.h declares, and fails loudly (no CPU fallback)
when no device is present.  CPU only (no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2411_01964_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "sqf2k_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sqf2k_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ["sqf2k_init", "sqf2k_primes", "sqf2k_sieve_bits", "sqf2k_scan_window",
                 "sqf2k_scan_exponents", "sqf2k_verify", "sqf2k_recheck",
                 "sqf2k_is_squarefree", "sqf2k_last_error", "sqf2k_shutdown"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header():
    # sqf2k_summary_t: 2 + 3*65 u64 + k_sum + n_failures + 2 u32
    assert ctypes.sizeof(_lib.Summary) == 8 * (2 + 3 * 65 + 2) + 8
    assert ctypes.sizeof(_lib.VerifyOpts) == 24
    assert _lib.load().sqf2k_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2411_01964_b200.runner import verify_range
    with pytest.raises(_lib.GPUError):
        verify_range(1, 1 << 10 | 1, 10)
    from paper_2411_01964_b200.primes import generate_primes
    with pytest.raises(_lib.GPUError):
        generate_primes(100)


def test_argument_errors_before_device():
    # validation mirrors the reference's ValueErrors and needs no device
    lib = _lib.load()
    s = _lib.Summary()
    assert lib.sqf2k_verify(4, 10, 3, None, ctypes.byref(s), None, 0) == _lib.EINVAL
    assert b"odd" in lib.sqf2k_last_error()
    assert lib.sqf2k_verify(3, 10, 3, None, ctypes.byref(s), None, 0) == _lib.EINVAL
    assert lib.sqf2k_verify(1, (1 << 62) + 3, 3, None, ctypes.byref(s), None, 0) == _lib.EINVAL
    assert lib.sqf2k_verify(1, 101, 0, None, ctypes.byref(s), None, 0) == _lib.EINVAL
    big = _lib.VerifyOpts(0, 0, (1 << 40) + 1, 0, 0)  # batch beyond the 32-bit tile counters' bound
    assert lib.sqf2k_verify(1, 101, 3, ctypes.byref(big), ctypes.byref(s), None, 0) == _lib.EINVAL
    assert b"batch_slots" in lib.sqf2k_last_error()
    deep = _lib.VerifyOpts(0, 17, 0, 0, 0)
    assert lib.sqf2k_verify(1, 101, 3, ctypes.byref(deep), ctypes.byref(s), None, 0) == _lib.EINVAL


def test_run_config_bounds():
    from paper_2411_01964_b200.runner import ConfigError, RunConfig
    with pytest.raises(ConfigError, match="batch_slots"):
        RunConfig(start=1, end=1 << 20, batch_slots=(1 << 40) + 1).validate()
    with pytest.raises(ConfigError, match="2\\^62"):
        RunConfig(start=1, end=(1 << 62) + 2).validate()
    with pytest.raises(ConfigError, match="tile_depth"):
        RunConfig(start=1, end=1 << 20, tile_depth=17).validate()
    with pytest.raises(ValueError, match="2\\^32"):
        from paper_2411_01964_b200.primes import generate_primes
        generate_primes(1 << 32)
