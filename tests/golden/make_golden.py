"""Generate the golden fixtures of tests/golden/ by running the REFERENCE
implementation itself (/root/reference/pkg/src/sqf2k, unmodified).

Run here (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # quick set  -> golden.json
    python tests/golden/make_golden.py --large    # + C2, 2^32, C3, 2^50 windows
                                                  #   -> golden_large.json (~5 min)

The reference package imports gmpy2 only for its heuristics module
(heuristics.py:22-24), which is absent from this image; an import-only stub
is put on sys.path after the reference (the hot path never calls it).  The
reference tree is read-only, so it is copied to a temp dir first.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import random
import shutil
import sys
import tempfile
import time
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

STUB = '''
class _Ctx:
    precision = 53
def get_context():
    return _Ctx()
def mpfr(*a, **k):
    raise NotImplementedError("gmpy2 import stub")
def rint(*a, **k):
    raise NotImplementedError("gmpy2 import stub")
'''


def import_reference():
    tmp = Path(tempfile.mkdtemp(prefix="sqf2k_ref_"))
    shutil.copytree(REF, tmp / "src")
    (tmp / "stub").mkdir()
    (tmp / "stub" / "gmpy2.py").write_text(STUB)
    sys.path[:0] = [str(tmp / "src"), str(tmp / "stub")]
    import sqf2k.aggregate as aggregate
    import sqf2k.primes as primes
    import sqf2k.runner as runner
    import sqf2k.search as search
    import sqf2k.sieve as sieve
    return primes, sieve, search, aggregate, runner


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def summary_json(s) -> dict:
    return {
        "start": s.start,
        "end": s.end,
        "histogram": {str(k): c for k, c in enumerate(s.histogram) if c},
        "k_sum": s.k_sum,
        "k_max_observed": s.k_max_observed,
        "record_candidates": {str(m): n for m, n in sorted(s.record_candidates.items())},
        "failures": list(s.failures),
    }


def quick(P, S, Q, A, R) -> dict:
    g: dict = {"source": "reference sqf2k 0.1.0 (/root/reference/pkg/src)"}

    # -- L0 prime table (test_primes.py) ------------------------------------
    g["prime_counts"] = {}
    g["prime_sha256"] = {}
    for lim in [1, 2, 3, 100, 3000, 4096, 37416, 10**5, 1 << 18, 1 << 20, (1 << 20) + 100]:
        t = P.generate_primes(lim)
        g["prime_counts"][str(lim)] = len(t)
        g["prime_sha256"][str(lim)] = sha(t.primes.astype("<i8").tobytes())
    g["primes_3000"] = P.generate_primes(3000).primes.tolist()

    # -- L1 segment sieve (test_sieve.py + random windows + near 2^50) ------
    p4 = P.generate_primes(10**4)
    p20 = P.generate_primes((1 << 20) + 100)
    p25 = P.generate_primes(1 << 25)
    cases = [
        (3, 33, 10**4), (1, 3, 10**4), (10**6 + 1, 10**6 + 2001, 10**4),
        (10**5 + 1, 10**5 + 80001, 10**4), (1, (1 << 14) + 1, 10**4),
        (101, 101 + (1 << 14), 10**4), (1, 129, 10**4), (1, 131, 10**4),
        ((1 << 39) + 1, (1 << 39) + 1 + (1 << 21), (1 << 20) + 100),
        ((1 << 50) - (1 << 22) + 1, (1 << 50) + 1, 1 << 25),
        ((1 << 50) - (1 << 20) - 1, (1 << 50) - 1, 1 << 25),
    ]
    rng = random.Random(0xB200)
    for _ in range(6):
        s = rng.randrange(1 << 20, 1 << 40) | 1
        w = rng.randrange(1, 1 << 12) * 2
        cases.append((s, s + w, (1 << 20) + 100))
    g["sieve"] = []
    for s, e, lim in cases:
        table = {10**4: p4, (1 << 20) + 100: p20, 1 << 25: p25}[lim]
        seg = S.sieve_segment(s, e, table)
        ent = {"start": s, "end": e, "prime_limit": lim, "sha256": sha(seg.bits.tobytes()),
               "nbytes": int(seg.bits.nbytes), "zeros": int((~seg.flags_bool()).sum())}
        if seg.bits.nbytes <= 4096:
            ent["hex"] = seg.bits.tobytes().hex()
        g["sieve"].append(ent)

    # -- L2 scan (test_search.py, test_aggregate.py) ------------------------
    p5 = P.generate_primes(10**5)
    p1m = P.generate_primes(1 << 20)

    def low(end):
        return Q.SegmentWindow(None, S.sieve_segment(1, end | 1, p5))

    g["scan"] = []

    def add_scan(name, window, k_max, with_kvals=True, **kw):
        summ = Q.scan_segment(window, k_max, **kw)
        ent = {"name": name, "k_max": k_max,
               "prev": None if window.previous is None else
               [window.previous.start, window.previous.end],
               "cur": [window.current.start, window.current.end],
               "summary": summary_json(summ)}
        if with_kvals:
            kv = Q.scan_exponents(window, k_max)
            ent["kvals_sha256"] = sha(kv.tobytes())
            if kv.nbytes <= 8192:
                ent["kvals_hex"] = kv.tobytes().hex()
        g["scan"].append(ent)

    add_scan("low_2^14_k13", low(1 << 14), 13)
    add_scan("low_2^14_k2", low(1 << 14), 2)
    add_scan("low_2^14_k1", low(1 << 14), 1)
    add_scan("low_2^15_k14", low(1 << 15), 14)
    add_scan("low_2^15_k14_b256", low(1 << 15), 14, block_slots=1 << 8)
    add_scan("low_2048_k10", low(2048), 10)
    add_scan("low_256_k1", low(256), 1)
    for seed in range(4):  # test_search.py:54-67
        r = random.Random(seed)
        start = r.randrange(1 << 20, 1 << 34) | 1
        w = Q.SegmentWindow(R.seed_predecessor(start, 14, p1m),
                            S.sieve_segment(start, start + (1 << 14), p1m))
        add_scan(f"high_seed{seed}_k14", w, 14)
    # shallow predecessor reaching 1, unaligned (search.py:120-125)
    for cs in [65, 101, 1001]:
        w = Q.SegmentWindow(S.sieve_segment(1, cs, p5), S.sieve_segment(cs, cs + 4000, p5))
        add_scan(f"shallow_prev_{cs}_k12", w, 12)
    # start=2^20+1 with k_max=8 predecessor (test_search.py:118-123)
    start = (1 << 20) + 1
    w = Q.SegmentWindow(R.seed_predecessor(start, 8, p5),
                        S.sieve_segment(start, start + (1 << 14), p5))
    add_scan("seeded_k8", w, 8)
    # near 2^50: 2^20-integer segment, k_max 16 (predecessor 2^15 slots)
    start = (1 << 50) - (1 << 20) + 1
    w = Q.SegmentWindow(R.seed_predecessor(start, 16, p25),
                        S.sieve_segment(start, (1 << 50) + 1, p25))
    add_scan("near2^50_k16", w, 16)
    # test_acceptance.py:199-223 windows (seed 0x51F2), kvals hashed
    rng = random.Random(0x51F2)
    width = 1 << 14
    for i in range(16):
        start = rng.randrange(1 << 20, (1 << 40) - width) | 1
        prev = R.seed_predecessor(start, 14, p20)
        cur = S.sieve_segment(start, start + width, p20)
        add_scan(f"accept_{i}_k14", Q.SegmentWindow(prev, cur), 14)
        rng.sample(range(width // 2), 625)  # keep the reference's rng stream

    # -- L4 run_verify reports ---------------------------------------------
    g["verify"] = []

    def add_verify(**cfg):
        t = time.time()
        rep = R.run_verify(R.RunConfig(**cfg))
        ent = {"config": cfg, "report_json": A.render_report_json(rep),
               "summary": summary_json(rep.summary),
               "counterexample_candidates": rep.counterexample_candidates,
               "seconds": round(time.time() - t, 3)}
        g["verify"].append(ent)
        print("verify", cfg, ent["seconds"], "s", file=sys.stderr)

    add_verify(start=1, end=1 << 20, segment_width=1 << 16)           # test_cli.py:21-42
    add_verify(start=3, end=16387, segment_width=1 << 14)              # README text example
    add_verify(start=1, end=1 << 24)                                   # C1
    add_verify(start=1, end=(1 << 20) + 1, segment_width=1 << 16, k_max=3)
    add_verify(start=1, end=1 << 18, segment_width=1 << 14, k_max=1)
    add_verify(start=1, end=1 << 18, segment_width=1 << 14, k_max=2)
    add_verify(start=(1 << 30) + 1, end=(1 << 30) + (1 << 22) + 7)
    add_verify(start=12345679, end=12345679 + 999999)
    add_verify(start=(1 << 40) - (1 << 21) + 1, end=1 << 40, segment_width=1 << 18)
    add_verify(start=(1 << 50) - (1 << 22) + 1, end=1 << 50, segment_width=1 << 20)
    add_verify(start=1, end=3 * (1 << 20) + 1, segment_width=1 << 20, k_max=20)  # README checkpoint
    add_verify(start=1, end=200_000_000)                               # test_acceptance.py:147
    return g


def large(R, A) -> dict:
    g = {"verify": []}
    cfgs = [
        dict(start=1, end=1_400_000_000),                      # C2
        dict(start=1, end=1 << 30),                            # Table 4
        dict(start=1, end=1 << 32),
        dict(start=(1 << 50) - (1 << 30) + 1, end=1 << 50),
        dict(start=(1 << 50) - (1 << 32) + 1, end=1 << 50),
        dict(start=1, end=1 << 36),                            # C3
        dict(start=(1 << 50) - (1 << 34) + 1, end=1 << 50),
    ]
    for cfg in cfgs:
        t = time.time()
        rep = R.run_verify(R.RunConfig(**cfg))
        ent = {"config": cfg, "report_json": A.render_report_json(rep),
               "summary": summary_json(rep.summary),
               "counterexample_candidates": rep.counterexample_candidates,
               "seconds": round(time.time() - t, 3)}
        g["verify"].append(ent)
        print("verify", cfg, ent["seconds"], "s", file=sys.stderr, flush=True)
    return g


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    args = ap.parse_args()
    P, S, Q, A, R = import_reference()
    if args.large:
        (OUT / "golden_large.json").write_text(json.dumps(large(R, A), indent=1) + "\n")
    else:
        (OUT / "golden.json").write_text(json.dumps(quick(P, S, Q, A, R), indent=1) + "\n")


if __name__ == "__main__":
    main()
