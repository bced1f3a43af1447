"""Host-side logic of the package (no GPU): summary merge algebra, record
finalisation, checkpoint format, report rendering and run configuration,
checked against the reference's golden outputs.  Mirrors the reference's
test_aggregate.py / test_acceptance.py host checks."""

import json

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2411_01964_b200.aggregate import (
    HIST_MAX_K,
    RecordTable,
    SegmentSummary,
    VerifyReport,
    finalize_records,
    merge,
    parse_checkpoint,
    read_checkpoint,
    render_bfile,
    render_report_csv,
    render_report_json,
    render_report_text,
    serialize_checkpoint,
    write_checkpoint,
)
from paper_2411_01964_b200.runner import ConfigError, RunConfig


@st.composite
def summary_in(draw, lo: int, hi: int) -> SegmentSummary:
    start = draw(st.integers(lo, hi - 4)) | 1
    end = draw(st.integers(start + 2, hi))
    end -= (end - start) % 2
    counts = draw(st.dictionaries(st.integers(1, 12), st.integers(0, 50), max_size=6))
    hist = [0] * (HIST_MAX_K + 1)
    for k, c in counts.items():
        hist[k] = c
    support = [k for k, c in enumerate(hist) if c]
    n_rec = draw(st.integers(0, 3))
    recs = {m: start + 2 * draw(st.integers(0, (end - start) // 2 - 1)) for m in range(1, n_rec + 1)}
    fails = sorted(draw(st.sets(st.integers(0, (end - start) // 2 - 1), max_size=3)))
    return SegmentSummary(start, end, hist, sum(k * c for k, c in enumerate(hist)),
                          max(support) if support else 0, recs, [start + 2 * i for i in fails])


triples = st.tuples(summary_in(1, 10**4), summary_in(10**4 + 1, 10**5), summary_in(10**5 + 1, 10**6))


@settings(max_examples=60, deadline=None)
@given(triples)
def test_merge_associative_commutative(t):
    a, b, c = t
    assert merge(merge(a, b), c) == merge(a, merge(b, c))
    assert merge(a, b) == merge(b, a)
    assert merge(SegmentSummary.empty(), a) == a


def test_merge_rejects_overlap():
    a = SegmentSummary(1, 101, [0] * 65, 0, 0, {}, [])
    b = SegmentSummary(51, 201, [0] * 65, 0, 0, {}, [])
    with pytest.raises(ValueError):
        merge(a, b)


def _summary_from_golden(g: dict) -> SegmentSummary:
    hist = [0] * (HIST_MAX_K + 1)
    for k, c in g["histogram"].items():
        hist[int(k)] = c
    return SegmentSummary(g["start"], g["end"], hist, g["k_sum"], g["k_max_observed"],
                          {int(m): n for m, n in g["record_candidates"].items()}, g["failures"])


def test_reports_render_byte_identical(golden):
    # the reference's final summaries, re-rendered by our host code
    for e in golden["verify"]:
        cfg = RunConfig(**e["config"])
        s = _summary_from_golden(e["summary"])
        s.validate()
        rep = VerifyReport(cfg.start, cfg.effective_end, cfg.segment_width, cfg.effective_k_max,
                           1, cfg.effective_end, 0.0, s,
                           counterexample_candidates=e["counterexample_candidates"])
        if cfg.start == 1 and not rep.counterexample_candidates:
            rep.records = finalize_records(s)
        assert render_report_json(rep) == e["report_json"], e["config"]
        csv = render_report_csv(rep)
        assert csv.splitlines()[0] == "section,key,value"
        assert "k_sum" in render_report_text(rep)


def test_finalize_records_rules():
    hist = [0] * 65
    hist[1] = 3
    s = SegmentSummary(1, 9, hist, 3, 1, {}, [])
    assert finalize_records(s).entries == {}
    with pytest.raises(ValueError):
        finalize_records(SegmentSummary(3, 9, hist, 3, 1, {}, []))  # not from 1
    with pytest.raises(ValueError):
        finalize_records(SegmentSummary(1, 11, hist, 3, 1, {}, []))  # gap
    with pytest.raises(ValueError):
        RecordTable({1: 29, 2: 11})  # not increasing
    assert render_bfile(RecordTable({1: 11, 2: 29})) == "1 11\n2 29\n"


def test_checkpoint_round_trip_and_corruption(tmp_path):
    # pkg/README.md:163-180 example
    text = ("sqf2k-checkpoint v1\nrange_start=1\nrange_end=67108865\nsegment_width=1048576\n"
            "k_max=20\nsequence=3\nnext_start=3145729\nelapsed_s=0.006629013998463051\n"
            "covered_start=1\ncovered_end=3145729\nk_sum=1912399\nk_max_observed=6\n"
            "histogram=1:1274906,2:259993,3:34588,4:3147,5:219,6:10\n"
            "records=1:11,2:29,3:533,4:849,5:434977\nfailures=\ncounterexamples=\nend\n")
    rep = parse_checkpoint(text)
    assert serialize_checkpoint(rep) == text
    assert not rep.complete and rep.summary.k_sum == 1912399
    p = tmp_path / "cp.txt"
    write_checkpoint(rep, p)
    assert p.read_text() == text and read_checkpoint(p) == rep
    assert not (tmp_path / "cp.txt.tmp").exists()
    for bad in [text.replace("sqf2k-checkpoint v1", "nope"), text[:-4], text.replace("k_sum", "ksum")]:
        with pytest.raises(ValueError):
            parse_checkpoint(bad)


def test_run_config_validation():
    for kw in [dict(start=4, end=100), dict(start=9, end=7), dict(end=100, segment_width=1000),
               dict(end=100, k_max=40), dict(end=100, workers=-1), dict(end=100, block_slots=100),
               dict(start=1, end=(1 << 62) + 2), dict(end=100, pipeline="tensor"),
               dict(end=100, tile_depth=17)]:
        with pytest.raises(ConfigError):
            RunConfig(**kw).validate()
    cfg = RunConfig(start=1, end=1 << 20)
    assert cfg.effective_end == (1 << 20) + 1 and cfg.effective_k_max == 30
    cfg.validate()


def test_golden_large_reports_render(golden_large):
    for e in golden_large["verify"]:
        cfg = RunConfig(**e["config"])
        s = _summary_from_golden(e["summary"])
        rep = VerifyReport(cfg.start, cfg.effective_end, cfg.segment_width, cfg.effective_k_max,
                           1, cfg.effective_end, 0.0, s)
        if cfg.start == 1:
            rep.records = finalize_records(s)
        assert render_report_json(rep) == e["report_json"], e["config"]
        doc = json.loads(e["report_json"])
        assert doc["odd_scanned"] == s.odd_scanned


def test_checkpoint_writer_keeps_order_and_surfaces_errors(tmp_path):
    # run_verify's background writer (batch-granular checkpoints): writes land
    # in submission order, the file holds the last one, errors reach the caller
    from paper_2411_01964_b200.aggregate import SegmentSummary, VerifyReport, read_checkpoint
    from paper_2411_01964_b200.runner import _CheckpointWriter

    path = tmp_path / "cp.txt"
    w = _CheckpointWriter(path)
    for seq in range(1, 6):
        w.submit(VerifyReport(start=1, end=1 << 20, segment_width=1 << 16, k_max=16, sequence=seq,
                              next_start=1 + seq * (1 << 16), elapsed_s=0.0,
                              summary=SegmentSummary.empty()))
    w.close()
    assert read_checkpoint(path).sequence == 5
    bad = _CheckpointWriter(tmp_path / "missing_dir" / "cp.txt")
    bad.submit(VerifyReport(start=1, end=3, segment_width=1 << 14, k_max=14, sequence=1,
                            next_start=3, elapsed_s=0.0, summary=SegmentSummary.empty()))
    with pytest.raises(OSError):
        bad.close()
