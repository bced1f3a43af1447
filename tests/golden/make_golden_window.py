"""Golden reports for the large windows (C4, C5) by PROCESS-SHARDED runs of
the unmodified reference (/root/reference/pkg/src/sqf2k).

    python tests/golden/make_golden_window.py --log2-width 40   # C4, ~10 min on 8 cores
    python tests/golden/make_golden_window.py --log2-width 44   # C5, ~2-3 h on 8 cores

The window [2^50 - 2^w + 1, 2^50) is cut into shards of 2^34 integers; each
shard is one `run_verify(RunConfig(s_i, s_{i+1}, workers=1))` of the
reference in its own process.  This is exactly the whole-window run
(SURVEY.md §8(c)): a run with start > 1 seeds its true predecessor
(reference runner.py:93-102), so every n in a shard is scanned against the
same bits as in one long run, and `merge` (aggregate.py:65-92) of summaries
over adjacent hulls is the segment loop's own reduction (runner.py:238).
The merged report is rendered by the reference's `render_report_json`
(aggregate.py:325-326) on `_as_report` of the full config (runner.py:285-297).

Shard results are appended to `<out>.partial.jsonl` as they finish, so an
interrupted generation resumes where it stopped.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import import_reference, summary_json  # noqa: E402

OUT = Path(__file__).resolve().parent
SHARD = 1 << 34
TOP = 1 << 50

_R = None


def _init():
    global _R
    _R = import_reference()


def _run_shard(bounds):
    s, e = bounds
    _P, _S, _Q, _A, R = _R
    t = time.time()
    rep = R.run_verify(R.RunConfig(start=s, end=e, workers=1))
    return {"start": s, "end": e, "summary": summary_json(rep.summary),
            "seconds": round(time.time() - t, 2)}


def shard_bounds(log2w: int) -> list[tuple[int, int]]:
    start = TOP - (1 << log2w) + 1
    out = []
    s = start
    while s < TOP:
        e = min(s + SHARD, TOP)
        out.append((s, e))
        s = e
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-width", type=int, required=True)
    ap.add_argument("--procs", type=int, default=8)
    args = ap.parse_args()
    w = args.log2_width
    out = OUT / f"golden_window_2p{w}.json"
    partial = OUT / f"golden_window_2p{w}.partial.jsonl"
    done = {}
    if partial.exists():
        for line in partial.read_text().splitlines():
            if line.strip():
                r = json.loads(line)
                done[r["start"]] = r
    todo = [b for b in shard_bounds(w) if b[0] not in done]
    print(f"{len(done)} shards done, {len(todo)} to go", file=sys.stderr, flush=True)
    t0 = time.time()
    with mp.get_context("fork").Pool(args.procs, initializer=_init) as pool, \
            partial.open("a") as f:
        for i, r in enumerate(pool.imap_unordered(_run_shard, todo)):
            f.write(json.dumps(r) + "\n")
            f.flush()
            done[r["start"]] = r
            print(f"[{i + 1}/{len(todo)}] shard {r['start']} {r['seconds']} s "
                  f"(elapsed {time.time() - t0:.0f} s)", file=sys.stderr, flush=True)

    P, S, Q, A, R = import_reference()
    cum = A.SegmentSummary.empty()
    for s, _e in shard_bounds(w):
        j = done[s]["summary"]
        hist = [0] * (A.HIST_MAX_K + 1)
        for k, c in j["histogram"].items():
            hist[int(k)] = c
        part = A.SegmentSummary(j["start"], j["end"], hist, j["k_sum"], j["k_max_observed"],
                                {int(m): n for m, n in j["record_candidates"].items()},
                                list(j["failures"]))
        part.validate()
        cum = A.merge(cum, part)
    cfg = R.RunConfig(start=TOP - (1 << w) + 1, end=TOP)
    assert cum.start == cfg.start and cum.end == cfg.effective_end
    assert cum.odd_scanned == A.odd_count(cfg.start, cfg.effective_end)
    assert not cum.failures  # k_max 30 never fails below 2^50
    n_seg = -(-(cfg.effective_end - cfg.start) // cfg.segment_width)
    rep = R._as_report(cfg, cum, n_seg, cfg.effective_end)
    g = {"source": "reference sqf2k 0.1.0 (/root/reference/pkg/src), process-sharded "
                   f"into {len(done)} runs of 2^34 integers, merged by aggregate.merge",
         "config": {"start": cfg.start, "end": cfg.end},
         "report_json": A.render_report_json(rep),
         "summary": summary_json(cum),
         "shard_seconds_total": round(sum(r["seconds"] for r in done.values()), 1)}
    out.write_text(json.dumps(g, indent=1) + "\n")
    print(f"wrote {out}", file=sys.stderr)


if __name__ == "__main__":
    main()
