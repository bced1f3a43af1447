"""TEST INFRASTRUCTURE ONLY -- ctypes front of the C restatement in
sqf2k_oracle.c (the parity checker and the CPU-baseline arm).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.  The product package
`paper_2411_01964_b200` never does; its GPU path fails loudly instead of
falling back here.

Return values mirror the reference's Python types so tests compare like
for like: prime tables are int64 numpy arrays (primes.py:11-16), segment
bits are padded uint8 arrays (sieve.py:19-25), summaries are dicts with the
SegmentSummary fields (aggregate.py:25-41).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "sqf2k_oracle.c"
LIB = HERE / "build" / "libsqf2k_oracle.so"
HIST_LEN = 65
NONE = (1 << 64) - 1


class Summary(ctypes.Structure):
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


def build(force: bool = False) -> Path:
    """Compile the restatement with gcc (seconds).  Idempotent."""
    if not force and LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(f".{os.getpid()}.tmp.so")
    subprocess.run(
        ["gcc", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread",
         "-o", str(tmp), str(SRC)],
        check=True,
    )
    os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = LIB if LIB.exists() else build()
        L = ctypes.CDLL(str(path))
        u64, u32, i64 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64
        vp = ctypes.c_void_p
        L.oracle_generate_primes.argtypes = [u64, vp, u64]
        L.oracle_generate_primes.restype = i64
        L.oracle_sieve_bits.argtypes = [u64, u64, vp, u64, u64, vp, u64]
        L.oracle_is_squarefree.argtypes = [u64, vp, u64]
        L.oracle_recheck.argtypes = [u64, vp, u64]
        L.oracle_scan_window.argtypes = [vp, u64, u64, vp, u64, u64, u32, u64,
                                         ctypes.POINTER(Summary), vp, u64]
        L.oracle_scan_exponents.argtypes = [vp, u64, u64, vp, u64, u64, u32, vp]
        L.oracle_verify.argtypes = [u64, u64, u64, u32, u64, ctypes.c_int,
                                    ctypes.POINTER(Summary), vp, u64]
        L.oracle_isqrt.argtypes = [u64]
        L.oracle_isqrt.restype = u64
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def generate_primes(limit: int) -> np.ndarray:
    """primes.py:26-40."""
    n = lib().oracle_generate_primes(limit, None, 0)
    if n == -1:
        raise ValueError(f"limit must be positive, got {limit}")
    out = np.empty(n, dtype=np.int64)
    lib().oracle_generate_primes(limit, _ptr(out), n)
    return out


def sieve_bits(start: int, end: int, primes: np.ndarray, limit: int) -> np.ndarray:
    """sieve.py:109-111 sieve_segment(...).bits"""
    n_slots = (end - start) // 2 if end > start else 0
    nbytes = ((n_slots + 63) // 64) * 8
    out = np.zeros(max(nbytes, 8), dtype=np.uint8)
    p = np.ascontiguousarray(primes, dtype=np.int64)
    rc = lib().oracle_sieve_bits(start, end, _ptr(p), len(p), limit, _ptr(out), nbytes)
    if rc:
        raise ValueError(f"bad sieve arguments [{start}, {end})")
    return out[:nbytes]


def is_squarefree(n: int, primes: np.ndarray) -> bool:
    p = np.ascontiguousarray(primes, dtype=np.int64)
    return bool(lib().oracle_is_squarefree(n, _ptr(p), len(p)))


def recheck(n: int, primes: np.ndarray) -> int | None:
    p = np.ascontiguousarray(primes, dtype=np.int64)
    k = lib().oracle_recheck(n, _ptr(p), len(p))
    return k or None


def summary_dict(s: Summary, failures: list[int]) -> dict:
    hist = [int(s.hist[k]) for k in range(HIST_LEN)]
    cand = {m: int(s.cand[m]) for m in range(1, HIST_LEN) if s.cand[m] != NONE}
    min_n = {k: int(s.min_n[k]) for k in range(1, HIST_LEN) if s.min_n[k] != NONE}
    return {
        "start": int(s.start),
        "end": int(s.end),
        "histogram": hist,
        "k_sum": int(s.k_sum),
        "k_max_observed": int(s.k_max_observed),
        "record_candidates": cand,
        "min_n": min_n,
        "failures": failures,
    }


def _call_with_failures(fn, cap: int = 1 << 12):
    while True:
        s = Summary()
        fail = np.zeros(max(cap, 1), dtype=np.uint64)
        rc = fn(ctypes.byref(s), _ptr(fail), cap)
        if rc == -4:
            cap = int(s.n_failures)
            continue
        if rc:
            raise ValueError(f"oracle rejected arguments (rc={rc})")
        return summary_dict(s, [int(x) for x in fail[: s.n_failures]])


def scan_window(prev: tuple[int, int, np.ndarray] | None,
                cur: tuple[int, int, np.ndarray], k_max: int,
                block_slots: int = 1 << 20) -> dict:
    """search.py:219-252 scan_segment over SegmentWindow(prev, cur)."""
    ps, pe, pb = prev if prev is not None else (0, 0, None)
    cs, ce, cb = cur
    return _call_with_failures(
        lambda s, f, cap: lib().oracle_scan_window(
            _ptr(pb), ps, pe, _ptr(cb), cs, ce, k_max, block_slots, s, f, cap))


def scan_exponents(prev, cur, k_max: int) -> np.ndarray:
    """search.py:255-279."""
    ps, pe, pb = prev if prev is not None else (0, 0, None)
    cs, ce, cb = cur
    out = np.zeros((ce - cs) // 2, dtype=np.uint8)
    rc = lib().oracle_scan_exponents(_ptr(pb), ps, pe, _ptr(cb), cs, ce, k_max, _ptr(out))
    if rc:
        raise ValueError("oracle rejected window")
    return out


def verify(start: int, end: int, *, width: int = 1 << 30, k_max: int | None = None,
           block_slots: int = 1 << 20, threads: int = 1) -> dict:
    """runner.py:216-252 merged segment-loop summary of [start, end) (end
    normalised as runner.py:57-61), before the k <= 63 failure recheck."""
    if (end - start) % 2:
        end += 1
    if k_max is None:
        k_max = width.bit_length() - 1
    return _call_with_failures(
        lambda s, f, cap: lib().oracle_verify(start, end, width, k_max, block_slots,
                                              threads, s, f, cap))


def odd_count(start: int, end: int) -> int:
    """aggregate.py:18-22"""
    return 0 if end <= start else end // 2 - start // 2


def verify_report(start: int, end: int, *, width: int = 1 << 30, k_max: int | None = None,
                  threads: int = 1) -> dict:
    """runner.py:172-282 for a complete run without checkpoint: the merged
    segment summary, failures rechecked to k <= 63 and folded into the
    histogram (runner.py:117-136, 258-276), records finalised for runs from 1
    (aggregate.py:121-143).  Returns report_dict's fields (aggregate.py:306-322)
    plus record_candidates."""
    if (end - start) % 2:
        end += 1
    if k_max is None:
        k_max = width.bit_length() - 1
    s = verify(start, end, width=width, k_max=k_max, threads=threads)
    hist = list(s["histogram"])
    failures = list(s["failures"])
    survivors = []
    if failures:
        primes = generate_primes(int(lib().oracle_isqrt(end - 1)))
        keep = []
        for n in failures:
            k = recheck(n, primes)
            if k is None:
                survivors.append(n)
                keep.append(n)
            else:
                hist[k] += 1
        failures = keep
    kmo = max([k for k, c in enumerate(hist) if c] or [0])
    records = None
    if start == 1 and not survivors:
        expected = odd_count(1, end) - 1
        assert sum(hist) + len(failures) == expected
        assert not failures
        entries = {m: n for m, n in s["record_candidates"].items() if 1 <= m < kmo}
        last = 0
        for m in sorted(entries):
            if entries[m] <= last:
                raise ValueError("record values must strictly increase with m")
            last = entries[m]
        records = [[m, entries[m]] for m in sorted(entries)]
    return {
        "range": {"start": start, "end": end},
        "odd_scanned": sum(hist) + len(failures),
        "histogram": [[k, c] for k, c in enumerate(hist) if k >= 1 and c > 0],
        "k_sum": sum(k * c for k, c in enumerate(hist)),
        "k_max_observed": kmo,
        "records": records,
        "failures": sorted(failures),
        "counterexample_candidates": survivors,
        "record_candidates": s["record_candidates"],
    }
