"""Parity of the CUDA path (through the C ABI / the reference-shaped Python
API) with the reference's golden vectors and with the oracle (the C
restatement, tests only).  Needs a B200: run with -m gpu."""

import hashlib
import json
import math
import random

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2411_01964_b200")
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.aggregate import render_report_json  # noqa: E402
from paper_2411_01964_b200.primes import generate_primes  # noqa: E402
from paper_2411_01964_b200.runner import RunConfig, run_verify, seed_predecessor, verify_range  # noqa: E402
from paper_2411_01964_b200.search import SegmentWindow, scan_exponents, scan_segment  # noqa: E402
from paper_2411_01964_b200.sieve import is_squarefree_oracle, sieve_segment  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module", autouse=True)
def native_loaded():
    L = _lib.lib()  # raises (no fallback) when the .so or the GPU is missing
    assert L.sqf2k_abi_version() == 1


# -- L0 primes -----------------------------------------------------------------

def test_prime_tables_match_golden(golden):
    for lim, count in golden["prime_counts"].items():
        t = generate_primes(int(lim))
        assert len(t) == count, lim
        assert t.primes.dtype == np.int64
        assert sha(t.primes.astype("<i8").tobytes()) == golden["prime_sha256"][lim], lim


def test_prime_tables_match_oracle():
    for lim in [2, 3, 4, 5, 8, 9, 10, 30, 31, 32, 33, 65535, 65536, 65537, (1 << 17) + 1,
                1 << 25, 33554393, 37416, 10**7]:
        t = generate_primes(lim)
        assert np.array_equal(t.primes, O.generate_primes(lim)), lim
    assert len(generate_primes(1 << 25)) == 2063689
    with pytest.raises(ValueError):
        generate_primes(0)
    assert len(generate_primes(1)) == 0


def test_prime_count_2_31():
    # pi(2^31) = 105097565 (the top of the GPU verifier's domain)
    assert len(generate_primes(1 << 31)) == 105097565


# -- L1 sieve ------------------------------------------------------------------

def test_sieve_matches_golden(golden):
    tables = {}
    for case in golden["sieve"]:
        lim = case["prime_limit"]
        if lim not in tables:
            tables[lim] = generate_primes(lim)
        seg = sieve_segment(case["start"], case["end"], tables[lim])
        assert seg.bits.nbytes == case["nbytes"]
        assert sha(seg.bits.tobytes()) == case["sha256"], (case["start"], case["end"])


def test_sieve_matches_oracle_random():
    rng = random.Random(7)
    p20 = generate_primes(1 << 20)
    p25 = generate_primes(1 << 25)
    cases = [(1, 3), (1, 5), (3, 5), (3, 33), (1, (1 << 20) + 1), (1, (1 << 21) + 1)]
    for _ in range(40):
        s = rng.randrange(1, 1 << 40) | 1
        w = rng.choice([2, 64, 126, 128, 130, 2048, 65534, 65536, 65538, 1 << 18, 3 << 17])
        cases.append((s, s + w))
    for _ in range(6):
        s = rng.randrange((1 << 50) - (1 << 30), 1 << 50) | 1
        cases.append((s, s + rng.choice([1 << 16, (1 << 20) + 2])))
    for s, e in cases:
        table = p20 if e <= (1 << 40) else p25
        want = O.sieve_bits(s, e, table.primes, table.limit)
        got = sieve_segment(s, e, table).bits
        assert np.array_equal(got, want), (s, e)


def test_sieve_large_segment_density():
    # test_sieve.py:47-53 at a full default-width segment near 2^50
    p25 = generate_primes(1 << 25)
    s = (1 << 50) - (1 << 30) + 1
    seg = sieve_segment(s, (1 << 50) + 1, p25)
    dens = np.unpackbits(seg.bits, bitorder="little")[: seg.n_slots].mean()
    assert abs(dens - 0.8106) < 0.001
    # spot-check against trial division
    rng = np.random.default_rng(3)
    idx = rng.integers(0, seg.n_slots, 64)
    ns = [s + 2 * int(i) for i in idx]
    for n in ns:
        assert seg.flag(n) == O.is_squarefree(n, p25.primes), n


def test_sieve_rejects_bad_ranges():
    p = generate_primes(10**4)
    for s, e in [(4, 10), (11, 11), (3, 10)]:
        with pytest.raises(ValueError):
            sieve_segment(s, e, p)
    with pytest.raises(ValueError):
        sieve_segment(3, 10**9, generate_primes(100))


def test_is_squarefree_oracle():
    p = O.generate_primes(1 << 20)
    rng = random.Random(11)
    for n in [1, 2, 4, 12, 27, 210, 1000003**2, (1 << 31) - 1] + \
             [rng.randrange(1, 1 << 32) for _ in range(200)]:
        assert is_squarefree_oracle(n) == O.is_squarefree(n, p), n
    with pytest.raises(ValueError):
        is_squarefree_oracle(0)


# -- L2 scan -------------------------------------------------------------------

def _gpu_window(entry, cache):
    def seg(s, e):
        lim = max(math.isqrt(e), 2)
        if lim not in cache:
            cache[lim] = generate_primes(lim)
        return sieve_segment(s, e, cache[lim])

    prev = seg(*entry["prev"]) if entry["prev"] else None
    return SegmentWindow(prev, seg(*entry["cur"]))


def test_scan_matches_golden(golden):
    cache = {}
    for entry in golden["scan"]:
        w = _gpu_window(entry, cache)
        s = scan_segment(w, entry["k_max"])
        want = entry["summary"]
        assert {str(k): c for k, c in enumerate(s.histogram) if c} == want["histogram"], entry["name"]
        assert s.k_sum == want["k_sum"]
        assert s.k_max_observed == want["k_max_observed"]
        assert {str(m): n for m, n in s.record_candidates.items()} == want["record_candidates"], entry["name"]
        assert s.failures == want["failures"], entry["name"]
        assert (s.start, s.end) == (want["start"], want["end"])
        kv = scan_exponents(w, entry["k_max"])
        assert sha(kv.tobytes()) == entry["kvals_sha256"], entry["name"]


def test_scan_matches_oracle_deep_windows():
    rng = random.Random(5)
    p25 = generate_primes(1 << 25)
    for k_max in [1, 2, 3, 7, 8, 9, 12, 16, 20, 24]:
        start = rng.randrange(1 << 30, 1 << 44) | 1
        prev = seed_predecessor(start, k_max, p25)
        cur = sieve_segment(start, start + rng.choice([1 << 12, 3 << 14, (1 << 18) + 6]), p25)
        w = SegmentWindow(prev, cur)
        got = scan_segment(w, k_max)
        want = O.scan_window((prev.start, prev.end, prev.bits), (cur.start, cur.end, cur.bits), k_max)
        assert got.histogram == want["histogram"], k_max
        assert got.record_candidates == want["record_candidates"], k_max
        assert got.failures == want["failures"], k_max
        kv = scan_exponents(w, k_max)
        assert np.array_equal(kv, O.scan_exponents((prev.start, prev.end, prev.bits),
                                                   (cur.start, cur.end, cur.bits), k_max))


def test_scan_window_errors():
    p = generate_primes(10**5)
    a = sieve_segment(1, (1 << 14) + 1, p)
    b = sieve_segment((1 << 14) + 3, (1 << 15) + 1, p)
    with pytest.raises(ValueError):
        SegmentWindow(a, b)
    w = SegmentWindow(None, sieve_segment(101, 101 + (1 << 14), p))
    with pytest.raises(ValueError):
        scan_exponents(w, 8)
    with pytest.raises(ValueError):
        scan_segment(w, 8)
    start = (1 << 20) + 1
    w = SegmentWindow(seed_predecessor(start, 8, p), sieve_segment(start, start + (1 << 14), p))
    with pytest.raises(ValueError):
        scan_exponents(w, 14)
    with pytest.raises(ValueError):
        scan_segment(w, 8, block_slots=100)


# -- L4 run_verify -------------------------------------------------------------

def _cfg(c):
    return RunConfig(**c)


@pytest.mark.parametrize("pipeline", ["fused", "bitmap"])
def test_run_verify_matches_golden_reports(golden, pipeline):
    for entry in golden["verify"]:
        cfg = _cfg(entry["config"])
        cfg.pipeline = pipeline
        rep = run_verify(cfg)
        assert render_report_json(rep) == entry["report_json"], entry["config"]
        want = entry["summary"]
        assert {str(m): n for m, n in rep.summary.record_candidates.items()} == \
            want["record_candidates"], entry["config"]


def test_run_verify_matches_large_goldens(golden_large):
    for entry in golden_large["verify"]:
        rep = run_verify(_cfg(entry["config"]))
        assert render_report_json(rep) == entry["report_json"], entry["config"]
        assert {str(m): n for m, n in rep.summary.record_candidates.items()} == \
            entry["summary"]["record_candidates"], entry["config"]


def test_paper_records_table3_to_2_36():
    # PAPER.md:274-285 / BASELINE.md: records m = 1..9 and hist of [1, 2^36)
    rep = run_verify(RunConfig(start=1, end=1 << 36))
    assert rep.records.entries == {1: 11, 2: 29, 3: 533, 4: 849, 5: 434977, 6: 10329791,
                                   7: 28819433, 8: 129747557, 9: 6915752957}
    assert rep.summary.odd_scanned == (1 << 35) - 1
    assert rep.summary.k_sum == 41776434485


def test_verify_matches_oracle_random_ranges():
    rng = random.Random(1234)
    for i in range(24):
        mag = rng.choice([20, 28, 34, 40, 46, 50])
        start = rng.randrange(1, 1 << mag) | 1
        width = rng.choice([2, 4, 130, 4096, 65536 * 2, (1 << 20) + 2, 3 << 19])
        end = start + width
        k_max = rng.choice([1, 2, 3, 5, 9, 13, 16, 17, 20, 30])
        want = O.verify(start, end, width=1 << 30, k_max=k_max)
        for pipeline, depth, batch, exact in [("fused", 0, 0, False), ("bitmap", 0, 0, False),
                                              ("fused", 4, 1 << 16, False),
                                              ("fused", 16, 3 << 16, True),
                                              ("bitmap", 6, 1 << 17, True)]:
            got = verify_range(start, end, k_max, pipeline=pipeline, tile_depth=depth,
                               batch_slots=batch, exact_buckets=exact)
            ctx = (start, end, k_max, pipeline, depth, batch, exact)
            assert got.histogram == want["histogram"], ctx
            assert got.record_candidates == want["record_candidates"], ctx
            assert got.failures == want["failures"], ctx
            assert got.k_sum == want["k_sum"]


def test_escalation_path_forced():
    # tile depth 1..3 forces most n through the exact trial-division kernel
    for depth in (1, 2, 3):
        for start, end, k_max in [(1, (1 << 16) + 1, 16), ((1 << 40) + 1, (1 << 40) + 20001, 12)]:
            want = O.verify(start, end, width=1 << 30, k_max=k_max)
            got = verify_range(start, end, k_max, tile_depth=depth)
            assert got.histogram == want["histogram"], (depth, start)
            assert got.record_candidates == want["record_candidates"]
            assert got.failures == want["failures"]


def test_batch_and_pipeline_invariance_large():
    end = (1 << 33) + 1
    base = verify_range(1, end, 30)
    for kw in [dict(batch_slots=1 << 28), dict(pipeline="bitmap"), dict(exact_buckets=True),
               dict(batch_slots=(1 << 26) + (1 << 16))]:
        got = verify_range(1, end, 30, **kw)
        assert got == base, kw
    # conservation: every odd n in (1, 2^33) counted once
    assert base.odd_scanned == (1 << 32) - 1


def test_recheck_matches_oracle():
    from paper_2411_01964_b200.runner import recheck_failures
    rng = random.Random(9)
    ns = [3, 5, 127, 849, 1 + 2**20] + [rng.randrange(3, 1 << 40) | 1 for _ in range(100)]
    p = O.generate_primes(1 << 20)
    assert recheck_failures(ns, 1 << 20) == [O.recheck(n, p) for n in ns]


def test_run_verify_failure_recheck_folds(golden):
    # k_max = 1: ~19 % of n fail the scan and are folded back by the recheck
    rep = run_verify(RunConfig(start=1, end=1 << 18, segment_width=1 << 14, k_max=1))
    want = [e for e in golden["verify"] if e["config"].get("k_max") == 1][0]
    assert render_report_json(rep) == want["report_json"]


def test_checkpoint_resume_byte_identical(tmp_path):
    # test_acceptance.py:241-254
    end, width = 1 << 22, 1 << 16
    golden = render_report_json(run_verify(RunConfig(start=1, end=end, segment_width=width)))
    for stop in (1, 13):
        cp = tmp_path / f"cp_{stop}.txt"
        cfg = RunConfig(start=1, end=end, segment_width=width, checkpoint_path=cp)
        part = run_verify(cfg, stop_after_segments=stop)
        assert not part.complete
        again = run_verify(cfg)
        assert again.complete
        assert render_report_json(again) == golden


def test_width_invariance():
    # test_acceptance.py:226-230
    golden = render_report_json(run_verify(RunConfig(start=1, end=1 << 30)))
    for width in (1 << 26, 1 << 28):
        assert render_report_json(run_verify(RunConfig(start=1, end=1 << 30, segment_width=width))) == golden


def test_acceptance_random_points():
    # test_acceptance.py:199-223: 16 windows below 2^40, seed 0x51F2
    rng = random.Random(0x51F2)
    width, k_max = 1 << 14, 14
    primes = generate_primes((1 << 20) + 100)
    table = O.generate_primes((1 << 20) + 100)
    for _ in range(16):
        start = rng.randrange(1 << 20, (1 << 40) - width) | 1
        w = SegmentWindow(seed_predecessor(start, k_max, primes), sieve_segment(start, start + width, primes))
        kv = scan_exponents(w, k_max)
        assert (kv > 0).all()
        flags = w.current.flags_bool()
        for i in rng.sample(range(width // 2), 625):
            n = start + 2 * i
            assert bool(flags[i]) == O.is_squarefree(n, table)
            k = next(k for k in range(1, 64) if O.is_squarefree(n - (1 << k), table))
            assert int(kv[i]) == k


def test_run_verify_errors():
    from paper_2411_01964_b200.runner import ConfigError
    with pytest.raises(ConfigError):
        run_verify(RunConfig(start=4, end=100))
    with pytest.raises(ConfigError):
        run_verify(RunConfig(start=1, end=(1 << 62) + 2))


@pytest.mark.parametrize("depth", [0, 10, 12])
def test_single_cta_long_runs(monkeypatch, depth):
    # one CTA walks many tiles, so the 4-quarter smem ring wraps repeatedly
    # and the first start phase of the t0 = 0 chunk drains an empty queue
    # (regression: a missing barrier let it drain stale shared memory)
    monkeypatch.setenv("SQF2K_DEBUG_GRID", "1")
    for lo, tiles in [(1, 13), ((1 << 33) + 1, 11), ((1 << 46) + 12345, 9)]:
        hi = lo + 2 * tiles * 65536 + 2 * 777
        want = O.verify(lo, hi, width=1 << 30, k_max=30)
        for _ in range(2):
            got = verify_range(lo, hi, 30, tile_depth=depth)
            assert got.histogram == want["histogram"], (lo, depth)
            assert got.k_sum == want["k_sum"]
            assert got.record_candidates == want["record_candidates"]


def test_paper_full_range_to_2_50():
    # the paper's whole computation: every odd 1 < n < 2^50,
    # ~40 s on one B200 -- k_sum, the maximal exponent 13 and Table 3
    s = verify_range(1, (1 << 50) + 1, 30)
    assert s.k_sum == 684465092067182
    assert s.k_max_observed == 13
    assert s.failures == []
    from paper_2411_01964_b200.aggregate import finalize_records
    rec = finalize_records(s).entries
    assert rec == {1: 11, 2: 29, 3: 533, 4: 849, 5: 434977, 6: 10329791, 7: 28819433,
                   8: 129747557, 9: 6915752957, 10: 2569472629649, 11: 23373845739407,
                   12: 60690478781437}


@pytest.mark.parametrize("grid", ["3", "5"])
def test_dynamic_chunks_against_oracle(monkeypatch, grid):
    # a handful of CTAs over hundreds of tiles: the static share, the
    # atomically handed-out chunks (each with its own halo pre-tile) and the
    # scheduler reset between launches all run, on both pipelines
    monkeypatch.setenv("SQF2K_DEBUG_GRID", grid)
    for lo, tiles in [(1, 400), ((1 << 44) + 3, 333)]:
        hi = lo + 2 * tiles * 65536 + 2 * 4321
        want = O.verify(lo, hi, width=1 << 30, k_max=30)
        for pipeline in ("fused", "bitmap"):
            for _ in range(2):
                got = verify_range(lo, hi, 30, pipeline=pipeline)
                assert got.histogram == want["histogram"], (lo, grid, pipeline)
                assert got.record_candidates == want["record_candidates"]


def test_top_of_domain_window():
    # the last odd n below 2^62 (the C ABI's domain end): primes up to 2^31,
    # every bucket class, products near 2^62 in u64
    hi = (1 << 62) - 1
    lo = hi - 2 * 600_000
    want = O.verify(lo, hi, width=1 << 30, k_max=30)
    for pipeline in ("fused", "bitmap"):
        got = verify_range(lo, hi, 30, pipeline=pipeline)
        assert got.histogram == want["histogram"], pipeline
        assert got.k_sum == want["k_sum"]
        assert got.record_candidates == want["record_candidates"]
        assert got.failures == want["failures"]


# -- C4 / C5: reports pinned to process-sharded reference runs -------------------

def _window_golden(log2w):
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", f"golden_window_2p{log2w}.json")
    if not os.path.exists(p):
        pytest.skip(f"golden_window_2p{log2w}.json not generated yet")
    return json.load(open(p))


@pytest.mark.parametrize("log2w", [40, 44])
def test_window_report_matches_reference(log2w):
    # C4 = [2^50 - 2^40 + 1, 2^50), C5 = [2^50 - 2^44 + 1, 2^50): the whole
    # report JSON (histogram, k_sum, odd_scanned, k_max_observed) against the
    # merged reference shards (tests/golden/make_golden_window.py)
    g = _window_golden(log2w)
    cfg = g["config"]
    for pipeline in (("fused", "bitmap") if log2w == 40 else ("fused",)):
        rep = run_verify(RunConfig(start=cfg["start"], end=cfg["end"], pipeline=pipeline))
        assert render_report_json(rep) == g["report_json"], pipeline
        want = g["summary"]
        assert {str(m): n for m, n in rep.summary.record_candidates.items()} == want["record_candidates"]


@pytest.mark.parametrize("log2w", [40, 44])
def test_window_shards_match_reference(log2w):
    # individual 2^34-integer reference runs (summaries incl. record candidates)
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", f"golden_window_2p{log2w}.partial.jsonl")
    if not os.path.exists(p):
        pytest.skip("no shard file")
    rows = [json.loads(x) for x in open(p).read().splitlines() if x.strip()]
    rng = random.Random(log2w)
    for r in rng.sample(rows, min(6, len(rows))):
        got = run_verify(RunConfig(start=r["start"], end=r["end"])).summary
        want = r["summary"]
        assert got.start == want["start"] and got.end == want["end"]
        assert {str(k): c for k, c in enumerate(got.histogram) if c} == want["histogram"]
        assert got.k_sum == want["k_sum"]
        assert {str(m): n for m, n in got.record_candidates.items()} == want["record_candidates"]
        assert got.failures == want["failures"]


def test_smallest_exponent_matches_scan_exponents():
    # search.py:66-90 scalar lookup against the GPU per-slot exponents and the
    # reference's known answers (test_search.py:25-31): 3, 5, 11, 29, 533, 849
    from paper_2411_01964_b200.search import smallest_exponent
    p = generate_primes(1 << 12)
    cur = sieve_segment(1, 1 << 12 | 1, p)
    w = SegmentWindow(None, cur)
    for n, k in [(3, 1), (5, 1), (11, 2), (29, 3), (533, 4), (849, 5), (127, 2)]:
        out = smallest_exponent(n, w, 12)
        assert out.found and out.k == k, (n, out)
    kv = scan_exponents(w, 12)
    rng = random.Random(11)
    for n in rng.sample(range(3, 1 << 12, 2), 200):
        out = smallest_exponent(n, w, 12)
        assert (out.k if out.found else 0) == int(kv[(n - 1) // 2]), n
    with pytest.raises(ValueError):
        smallest_exponent(4, w, 12)
    with pytest.raises(ValueError):
        smallest_exponent(11, w, 0)


def test_pattern13_table_batches():
    # the p = 3..13 wheel table (kind 2, tile.cuh) serves fused calls from
    # 2^28 slots, the p <= 11 one (kind 1) the rest; SQF2K_DEBUG_PAT13_MIN
    # moves the threshold, so the same windows run once on each kind -- every
    # batch reading the wheel table at its own word offset (wheel_offset,
    # tile.cu) -- and must agree (both are pinned to the reference's reports
    # by test_run_verify_matches_large_goldens).
    import os
    import subprocess
    import sys
    code = (
        "import json, sys\n"
        "from paper_2411_01964_b200.runner import verify_range\n"
        "s, e = (1 << 50) - (1 << 34) + 1, (1 << 50) + 1\n"
        "out = [verify_range(s, e, 30, batch_slots=b) for b in (0, 1 << 30, 1 << 28, (1 << 28) + 32)]\n"
        "out += [verify_range(1, (1 << 33) + 1, 30, batch_slots=1 << 27)]\n"
        "out += [verify_range(s0, s0 + (1 << 22), 30) for s0 in (3, (1 << 40) + 7, (1 << 45) + 12345)]\n"
        "print(json.dumps([[o.histogram, o.k_sum, sorted(o.record_candidates.items())] for o in out]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    got = {}
    for kind, lim in (("kind2", "0"), ("kind1", str(1 << 62))):
        r = subprocess.run([sys.executable, "-c", code], cwd=root,
                           env=dict(os.environ, SQF2K_DEBUG_PAT13_MIN=lim), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        got[kind] = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["kind2"] == got["kind1"]
    for g in got["kind2"][1:4]:
        assert g == got["kind2"][0]
    want = verify_range((1 << 50) - (1 << 34) + 1, (1 << 50) + 1, 30)
    assert got["kind2"][0] == [want.histogram, want.k_sum,
                               [list(x) for x in sorted(want.record_candidates.items())]]


@pytest.mark.parametrize("item,bias", [("3", "0"), ("16", "0.25"), ("20", "0.5")])
def test_medium_schedules_agree(item, bias):
    # every medium-prime schedule (build_med's knobs, read from the
    # environment) must give the same result; items 16 and 20 once hung the
    # tile kernel (a warp split across two phases, fixed by a warp-uniform
    # `need`), so the subprocess runs under a timeout
    import os
    import subprocess
    import sys
    code = (
        "import json\n"
        "from paper_2411_01964_b200.runner import verify_range\n"
        "out = [verify_range((1 << 50) - (1 << 32) + 1, (1 << 50) + 1, 30),\n"
        "       verify_range(1, (1 << 31) + 1, 30), verify_range(1, (1 << 28) + 1, 30)]\n"
        "print(json.dumps([[o.histogram, o.k_sum, sorted(o.record_candidates.items())] for o in out]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SQF2K_MED_ITEM=item, SQF2K_MED_BIAS=bias)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    want = [verify_range((1 << 50) - (1 << 32) + 1, (1 << 50) + 1, 30), verify_range(1, (1 << 31) + 1, 30),
            verify_range(1, (1 << 28) + 1, 30)]
    assert got == [[w.histogram, w.k_sum, [list(x) for x in sorted(w.record_candidates.items())]] for w in want]


def test_domain_top_large_window():
    # a 2^40-integer window just below 2^62 (the domain's top): bucket primes
    # up to 2^31 with q = p^2 near 2^62, where u0 + 4q passes 2^64 -- the
    # bucket pass once counted such wrapped positions as hits (an illegal
    # address); pipelines, bucket modes and batch sizes must agree, and
    # every odd n must be counted once
    s, e = (1 << 62) - (1 << 40) + 1, (1 << 62) - 1
    base = verify_range(s, e, 30)
    assert base.odd_scanned == (e - s) // 2
    assert not base.failures
    for kw in [dict(pipeline="bitmap"), dict(exact_buckets=True), dict(batch_slots=1 << 36)]:
        assert verify_range(s, e, 30, **kw) == base, kw
