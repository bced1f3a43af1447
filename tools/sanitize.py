"""Small ranges through every kernel of the hot path, for compute-sanitizer
(memcheck / racecheck / synccheck on small ranges).

    compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize.py

Covers the fused tile kernel and the export (bitmap) pipeline with the
split-phase mbarrier ring at the default grid and with 1 and 3 CTAs (long
per-CTA runs, dynamic chunks), the window scan kernels, the prime
generators, escalation, recheck and trial division -- on [1, 2^20] and on a
2^20-integer window ending at 2^50 -- plus the dense bucket pass and the
per-call p <= 13 pattern table on a 2^32-integer window.  Results are checked against the oracle
so a sanitizer run is also a parity run.
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("SQF2K_NO_GRAPHS", "1")


def main() -> None:
    from oracle import oracle as O
    from paper_2411_01964_b200.primes import generate_primes
    from paper_2411_01964_b200.runner import recheck_failures, verify_range
    from paper_2411_01964_b200.search import SegmentWindow, scan_exponents, scan_segment
    from paper_2411_01964_b200.sieve import is_squarefree_oracle, sieve_segment
    from paper_2411_01964_b200.runner import seed_predecessor

    ranges = [(1, (1 << 20) + 1), ((1 << 50) - (1 << 20) + 1, (1 << 50) + 1)]
    grids = [None, "1", "3"]
    for lo, hi in ranges:
        want = O.verify(lo, hi, width=1 << 30, k_max=30)
        for grid in grids:
            if grid is None:
                os.environ.pop("SQF2K_DEBUG_GRID", None)
            else:
                os.environ["SQF2K_DEBUG_GRID"] = grid
            for pipeline in ("fused", "bitmap"):
                for depth in (0, 4):  # default depth, and forced escalation
                    got = verify_range(lo, hi, 30, pipeline=pipeline, tile_depth=depth)
                    assert got.histogram == want["histogram"], (lo, grid, pipeline, depth)
                    assert got.record_candidates == want["record_candidates"]
            print(f"verify [{lo}, {hi}) grid {grid}: ok", flush=True)
    os.environ.pop("SQF2K_DEBUG_GRID", None)
    # a 2^32-integer window at 2^50 in one batch: the tile-major dense bucket
    # pass; then the same window with the per-call p <= 13 pattern table in a
    # child process (SQF2K_DEBUG_PAT13_MIN is read once per process), in one
    # batch and in two
    import json
    import subprocess
    big = ((1 << 50) - (1 << 32) + 1, (1 << 50) + 1)
    want = verify_range(*big, 30, batch_slots=1 << 31)
    code = ("import json, sys\n"
            f"sys.path.insert(0, {str(ROOT)!r})\n"
            "from paper_2411_01964_b200.runner import verify_range\n"
            f"out = [verify_range({big[0]}, {big[1]}, 30, batch_slots=b) for b in (1 << 31, 1 << 30)]\n"
            "print(json.dumps([[o.histogram, sorted(o.record_candidates.items())] for o in out]))\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SQF2K_DEBUG_PAT13_MIN="0"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    for h, c in json.loads(r.stdout.strip().splitlines()[-1]):
        assert h == want.histogram and c == [list(x) for x in sorted(want.record_candidates.items())]
    print(f"verify [{big[0]}, {big[1]}) dense buckets, p <= 13 table: ok", flush=True)
    # k_max = 2: failures, the failure sort and the recheck kernel
    got = verify_range(1, (1 << 16) + 1, 2)
    want = O.verify(1, (1 << 16) + 1, width=1 << 30, k_max=2)
    assert got.failures == want["failures"]
    ks = recheck_failures(got.failures[:64], 256)
    assert all(k is not None for k in ks)
    # prime tables: the one-CTA generator and the segmented one
    for lim in (1000, 1 << 20, (1 << 25) + 7):
        assert len(generate_primes(lim)) == len(O.generate_primes(lim))
    # sieve_segment export and the window scans (scan_segment, scan_exponents)
    p25 = generate_primes(1 << 25)
    start = (1 << 50) - (1 << 20) + 1
    w = SegmentWindow(seed_predecessor(start, 16, p25), sieve_segment(start, (1 << 50) + 1, p25))
    s = scan_segment(w, 16)
    k = scan_exponents(w, 16)
    assert s.odd_scanned == len(k)
    n = (1 << 40) | 1
    assert is_squarefree_oracle(n) == O.is_squarefree(n, O.generate_primes(1 << 20))
    print("sanitize run: all kernels ok", flush=True)


if __name__ == "__main__":
    main()
