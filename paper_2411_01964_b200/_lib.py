"""ctypes binding of libsqf2k_b200.so (declared in include/sqf2k_b200.h).

There is no CPU fallback: if the in-tree library is missing, or no CUDA
device is visible, every hot-path call raises.  Errors cross the C ABI as
negative codes and are mapped here onto the exceptions the reference raises
(ValueError for bad arguments, sieve.py:80-88 / search.py:233-236 style).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

# SQF2K_LIB: an alternative build of the same library (debug / checks
# variants, tools/build_exp.sh); default the in-tree build
LIB_PATH = Path(os.environ.get("SQF2K_LIB") or Path(__file__).resolve().parent / "libsqf2k_b200.so")

HIST_LEN = 65
NONE = (1 << 64) - 1

OK, EINVAL, ECUDA, ENOMEM, ECAPACITY, ENODEV = 0, -1, -2, -3, -4, -5


class Summary(ctypes.Structure):
    """sqf2k_summary_t"""

    _fields_ = [
        ("start", ctypes.c_uint64),
        ("end", ctypes.c_uint64),
        ("hist", ctypes.c_uint64 * HIST_LEN),
        ("min_n", ctypes.c_uint64 * HIST_LEN),
        ("cand", ctypes.c_uint64 * HIST_LEN),
        ("k_sum", ctypes.c_uint64),
        ("n_failures", ctypes.c_uint64),
        ("k_max_observed", ctypes.c_uint32),
        ("k_max", ctypes.c_uint32),
    ]


class VerifyOpts(ctypes.Structure):
    """sqf2k_verify_opts_t"""

    _fields_ = [
        ("pipeline", ctypes.c_uint32),
        ("tile_depth", ctypes.c_uint32),
        ("batch_slots", ctypes.c_uint64),
        ("flags", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]


EXACT_BUCKETS = 1


class KStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64),
                ("total_ms", ctypes.c_double)]


# every symbol include/sqf2k_b200.h declares: name -> (restype, argtypes)
_u64, _u32, _i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
_vp = ctypes.c_void_p
SIGNATURES = {
    "sqf2k_init": (_i32, [_i32]),
    "sqf2k_device_count": (_i32, [ctypes.POINTER(_i32)]),
    "sqf2k_last_error": (ctypes.c_char_p, []),
    "sqf2k_shutdown": (None, []),
    "sqf2k_abi_version": (_i32, []),
    "sqf2k_prime_count": (_i32, [_u64, ctypes.POINTER(_u64)]),
    "sqf2k_primes": (_i32, [_u64, _vp, _u64, ctypes.POINTER(_u64)]),
    "sqf2k_sieve_bits": (_i32, [_u64, _u64, _vp, _u64, _vp, _u64]),
    "sqf2k_scan_window": (_i32, [_vp, _u64, _u64, _vp, _u64, _u64, _u32,
                                 ctypes.POINTER(Summary), _vp, _u64]),
    "sqf2k_scan_exponents": (_i32, [_vp, _u64, _u64, _vp, _u64, _u64, _u32, _vp, _u64]),
    "sqf2k_verify": (_i32, [_u64, _u64, _u32, ctypes.POINTER(VerifyOpts),
                            ctypes.POINTER(Summary), _vp, _u64]),
    "sqf2k_recheck": (_i32, [_vp, _u64, _u64, _vp]),
    "sqf2k_is_squarefree": (_i32, [_vp, _u64, _u64, _vp]),
    "sqf2k_profile_enable": (_i32, [_i32]),
    "sqf2k_profile_reset": (_i32, []),
    "sqf2k_profile_read": (_i32, [ctypes.POINTER(KStat), _i32, ctypes.POINTER(_i32)]),
    "sqf2k_sync": (_i32, []),
    "sqf2k_stream": (_vp, []),
    "sqf2k_copy_stats": (_i32, [ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None
_device: int | None = None


class GPUError(RuntimeError):
    """A CUDA-side failure of the hot path (no CPU fallback exists)."""


def load() -> ctypes.CDLL:
    """Load the in-tree library (no device needed).  Raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is not built; run `python -m paper_2411_01964_b200.build` "
                    "(the B200 path has no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def _raise(rc: int) -> None:
    msg = (load().sqf2k_last_error() or b"").decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise GPUError(f"libsqf2k_b200 error {rc}: {msg}")


def check(rc: int) -> None:
    if rc != OK:
        _raise(rc)


def default_device() -> int:
    for key in ("SQF2K_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


def lib() -> ctypes.CDLL:
    """The library bound to this process's GPU (initialised on first use)."""
    global _device
    L = load()
    if _device is None:
        dev = default_device()
        check(L.sqf2k_init(dev))
        _device = dev
    return L


def bound_device() -> int:
    """The CUDA device this process's library is bound to (binds it if needed)."""
    lib()
    return int(_device)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def profile(enable: bool) -> None:
    check(lib().sqf2k_profile_enable(1 if enable else 0))


def profile_reset() -> None:
    check(lib().sqf2k_profile_reset())


def profile_read() -> dict[str, tuple[int, float]]:
    """{kernel name: (launches, total device ms)} since the last reset."""
    L = lib()
    n = ctypes.c_int(0)
    check(L.sqf2k_profile_read(None, 0, ctypes.byref(n)))
    buf = (KStat * max(n.value, 1))()
    check(L.sqf2k_profile_read(buf, n.value, ctypes.byref(n)))
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms))
            for i in range(n.value)}


def copy_stats() -> tuple[int, int]:
    """(host->device, device->host) bytes copied since the last profile reset."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(lib().sqf2k_copy_stats(ctypes.byref(a), ctypes.byref(b)))
    return int(a.value), int(b.value)


def stream_handle() -> int:
    """The library's cudaStream_t as an integer (for torch.cuda.ExternalStream)."""
    return int(lib().sqf2k_stream() or 0)


def sync() -> None:
    check(lib().sqf2k_sync())
