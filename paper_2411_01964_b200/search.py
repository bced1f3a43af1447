"""L2 smallest-exponent search (mirror of sqf2k.search,
/root/reference/pkg/src/sqf2k/search.py).

`scan_segment` / `scan_exponents` upload the two-segment window once and run
the 128-slot-per-thread scan kernel of csrc/scan.cu: flags of n - 2^k for
consecutive odd n are the window bits shifted by 2^(k-1) slots, read with
funnel shifts (k <= 8) or aligned 128-bit loads (k >= 9).  The block plan
and worker count of the reference only partition the work, so they are
validated and otherwise ignored: results are identical by the merge law
(search.py:24-27).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_2411_01964_b200 import _lib
from paper_2411_01964_b200.aggregate import HIST_MAX_K, SegmentSummary, from_device
from paper_2411_01964_b200.sieve import Segment

FOUND = "FOUND"
NOT_FOUND = "NOT_FOUND"
DEFAULT_BLOCK_SLOTS = 1 << 20


@dataclass(frozen=True)
class SegmentWindow:
    """Current segment plus its predecessor (search.py:30-51)."""

    previous: Segment | None
    current: Segment

    def __post_init__(self) -> None:
        if self.previous is not None and self.previous.end != self.current.start:
            raise ValueError(
                f"segments not adjacent: previous ends at {self.previous.end}, "
                f"current starts at {self.current.start}")

    def flag(self, m: int) -> bool:
        if m >= self.current.start:
            return self.current.flag(m)
        if self.previous is None:
            raise ValueError(f"{m} is below the window (no predecessor)")
        return self.previous.flag(m)


@dataclass(frozen=True)
class SearchOutcome:
    n: int
    status: str
    k: int | None = None
    m: int | None = None

    @property
    def found(self) -> bool:
        return self.status == FOUND


def smallest_exponent(n: int, window: SegmentWindow, k_max: int) -> SearchOutcome:
    """Scalar lookup of one n in an already-sieved window (search.py:66-90);
    a debugging aid that reads window bits, not a compute path."""
    cur = window.current
    if n % 2 == 0 or not (cur.start <= n < cur.end):
        raise ValueError(f"{n} is not an odd member of [{cur.start}, {cur.end})")
    if k_max < 1:
        raise ValueError(f"k_max must be positive, got {k_max}")
    low = window.previous.start if window.previous is not None else cur.start
    for k in range(1, k_max + 1):
        m = n - (1 << k)
        if m < 1:
            break
        if m < low:
            raise ValueError(
                f"lookup {m} = {n} - 2^{k} falls below the window at {low}; "
                f"k_max {k_max} exceeds what this window supports")
        if window.flag(m):
            return SearchOutcome(n, FOUND, k, m)
    return SearchOutcome(n, NOT_FOUND)


def _window_args(window: SegmentWindow):
    prev = window.previous
    cur = window.current
    pb = None if prev is None else np.ascontiguousarray(prev.bits)
    cb = np.ascontiguousarray(cur.bits)
    return (pb, 0 if prev is None else prev.start, 0 if prev is None else prev.end,
            cb, cur.start, cur.end)


def scan_segment(window: SegmentWindow, k_max: int, *, block_slots: int = DEFAULT_BLOCK_SLOTS,
                 workers: int = 1) -> SegmentSummary:
    """Histogram, k_sum, records candidates and failures of the current
    segment (search.py:219-252), computed on the GPU."""
    if k_max < 1:
        raise ValueError(f"k_max must be positive, got {k_max}")
    if block_slots < 64 or block_slots % 64:
        raise ValueError("block_slots must be a positive multiple of 64")
    if k_max > HIST_MAX_K - 1:
        raise ValueError(f"k_max {k_max} beyond 63")
    pb, ps, pe, cb, cs, ce = _window_args(window)
    L = _lib.lib()
    cap = 1 << 12
    while True:
        s = _lib.Summary()
        fail = np.zeros(cap, dtype=np.uint64)
        rc = L.sqf2k_scan_window(_lib.ptr(pb), ps, pe, _lib.ptr(cb), cs, ce, k_max,
                                 ctypes.byref(s), _lib.ptr(fail), cap)
        if rc == _lib.ECAPACITY:
            cap = int(s.n_failures)
            continue
        _lib.check(rc)
        return from_device(s, fail[: s.n_failures].tolist())


def scan_exponents(window: SegmentWindow, k_max: int) -> np.ndarray:
    """Per-slot smallest exponents of the current segment, 0 when unresolved
    or n = 1 (search.py:255-279), computed on the GPU."""
    if k_max < 1:
        raise ValueError(f"k_max must be positive, got {k_max}")
    pb, ps, pe, cb, cs, ce = _window_args(window)
    n_slots = window.current.n_slots
    out = np.zeros(n_slots, dtype=np.uint8)
    _lib.check(_lib.lib().sqf2k_scan_exponents(_lib.ptr(pb), ps, pe, _lib.ptr(cb), cs, ce,
                                               k_max, _lib.ptr(out), n_slots))
    return out
