"""Pin the oracle (C restatement, test infrastructure) to the reference:
golden vectors produced by the reference itself (tests/golden/make_golden.py)
and the known answers in the reference's own tests.  CPU only."""

import hashlib
import json

import numpy as np
import pytest

from oracle import oracle as O


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def hist_dict(h):
    return {str(k): c for k, c in enumerate(h) if c}


def test_prime_counts_and_tables(golden):
    for lim, count in golden["prime_counts"].items():
        t = O.generate_primes(int(lim))
        assert len(t) == count, lim
        assert sha(t.astype("<i8").tobytes()) == golden["prime_sha256"][lim], lim
    assert O.generate_primes(3000).tolist() == golden["primes_3000"]
    # test_primes.py:27-38
    assert len(O.generate_primes(100)) == 25
    assert len(O.generate_primes(10**5)) == 9592
    assert O.generate_primes(2).tolist() == [2]
    assert len(O.generate_primes(1)) == 0
    with pytest.raises(ValueError):
        O.generate_primes(0)


def test_sieve_segments(golden):
    tables = {}
    for case in golden["sieve"]:
        lim = case["prime_limit"]
        if lim not in tables:
            tables[lim] = O.generate_primes(lim)
        bits = O.sieve_bits(case["start"], case["end"], tables[lim], lim)
        assert bits.nbytes == case["nbytes"]
        assert sha(bits.tobytes()) == case["sha256"], (case["start"], case["end"])


def test_sieve_known_answers():
    p = O.generate_primes(10**4)
    bits = O.sieve_bits(3, 33, p, 10**4)  # test_sieve.py:19-22
    flags = np.unpackbits(bits, bitorder="little")[:15]
    assert {3 + 2 * i for i in range(15) if not flags[i]} == {9, 25, 27}
    with pytest.raises(ValueError):
        O.sieve_bits(4, 10, p, 10**4)
    with pytest.raises(ValueError):
        O.sieve_bits(3, 10, p, 10**4)
    with pytest.raises(ValueError):
        O.sieve_bits(3, 10**9, O.generate_primes(100), 100)


def _window(entry, tables):
    def seg(s, e):
        lim = int(np.sqrt(e)) + 2
        if lim not in tables:
            tables[lim] = O.generate_primes(lim)
        return (s, e, O.sieve_bits(s, e, tables[lim], lim))

    prev = seg(*entry["prev"]) if entry["prev"] else None
    return prev, seg(*entry["cur"])


def test_scan_windows(golden):
    tables = {}
    for entry in golden["scan"]:
        prev, cur = _window(entry, tables)
        got = O.scan_window(prev, cur, entry["k_max"])
        want = entry["summary"]
        assert hist_dict(got["histogram"]) == want["histogram"], entry["name"]
        assert got["k_sum"] == want["k_sum"]
        assert got["k_max_observed"] == want["k_max_observed"]
        assert {str(m): n for m, n in got["record_candidates"].items()} == want["record_candidates"]
        assert got["failures"] == want["failures"], entry["name"]
        kv = O.scan_exponents(prev, cur, entry["k_max"])
        assert sha(kv.tobytes()) == entry["kvals_sha256"], entry["name"]


def test_scan_known_answers():
    p = O.generate_primes(10**5)
    cur = (1, 2049, O.sieve_bits(1, 2049, p, 10**5))
    kv = O.scan_exponents(None, cur, 10)
    for n, k in [(3, 1), (5, 1), (11, 2), (29, 3), (533, 4), (849, 5), (127, 2)]:
        assert kv[(n - 1) // 2] == k, n  # test_search.py:26-32
    cur = (1, (1 << 14) + 1, O.sieve_bits(1, (1 << 14) + 1, p, 10**5))
    s = O.scan_window(None, cur, 13)  # test_search.py:70-79
    assert sum(s["histogram"]) == 8191 and s["failures"] == []
    assert [s["record_candidates"][m] for m in (1, 2, 3, 4)] == [11, 29, 533, 849]


def test_verify_reports(golden):
    for entry in golden["verify"]:
        cfg = dict(entry["config"])
        kw = {}
        if "segment_width" in cfg:
            kw["width"] = cfg["segment_width"]
        if "k_max" in cfg:
            kw["k_max"] = cfg["k_max"]
        rep = O.verify_report(cfg["start"], cfg["end"], threads=4, **kw)
        want = json.loads(entry["report_json"])
        for key in ("range", "odd_scanned", "histogram", "k_sum", "k_max_observed",
                    "records", "failures", "counterexample_candidates"):
            assert rep[key] == want[key], (cfg, key)
        assert {str(m): n for m, n in rep["record_candidates"].items()} == \
            entry["summary"]["record_candidates"], cfg


def test_verify_thread_invariance():
    a = O.verify(1, 1 << 22, width=1 << 16, threads=1)
    b = O.verify(1, 1 << 22, width=1 << 16, threads=7)
    c = O.verify(1, 1 << 22, width=1 << 18, threads=3)
    assert a == b
    for key in ("histogram", "k_sum", "record_candidates", "failures", "min_n"):
        assert a[key] == c[key]


def test_acceptance_known_answers(golden):
    # test_cli.py:32-42 and test_stats.py:63: [1, 2^20]
    rep = O.verify_report(1, 1 << 20, width=1 << 16)
    assert rep["odd_scanned"] == 524287 and rep["k_sum"] == 637484
    assert dict(map(tuple, rep["records"])) == {1: 11, 2: 29, 3: 533, 4: 849, 5: 434977}
    assert dict(map(tuple, rep["histogram"])) == {1: 424973, 2: 86638, 3: 11544, 4: 1059, 5: 71, 6: 2}
    # test_acceptance.py:36-45 records to 2e8
    rep = O.verify_report(1, 200_000_000, threads=8)
    assert dict(map(tuple, rep["records"])) == {
        1: 11, 2: 29, 3: 533, 4: 849, 5: 434977, 6: 10329791, 7: 28819433, 8: 129747557}


@pytest.mark.slow
def test_large_goldens(golden_large):
    for entry in golden_large["verify"]:
        cfg = entry["config"]
        if cfg["end"] - cfg["start"] > (1 << 33):
            continue
        rep = O.verify_report(cfg["start"], cfg["end"], threads=8)
        want = json.loads(entry["report_json"])
        assert rep["histogram"] == want["histogram"]
        assert rep["k_sum"] == want["k_sum"]
        assert rep["records"] == want["records"]
