"""Reproduce the paper's full computation on one GPU: every odd 1 < n < 2^50
(PAPER.md:258-301).  Checks k_sum = 684465092067182, max k = 13 and the
Table 3 records, and prints the timing.   python tools/full_2p50.py [LOG2]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.aggregate import finalize_records  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 50
end = (1 << log2) + 1
verify_range(1, (1 << 30) + 1, 30)  # warm-up: buffers, tables
_lib.sync()
from bench import ClockSampler  # noqa: E402  (nvidia-smi clocks during the run)
clocks = ClockSampler(_lib.bound_device()).__enter__()
t = time.perf_counter()
s = verify_range(1, end, 30)
dt = time.perf_counter() - t
clocks.__exit__(None, None, None)
rec = finalize_records(s).entries
out = {"range": [1, end], "odd_n": (end - 1) // 2 - 1, "seconds": dt,
       "odd_n_per_s": ((end - 1) // 2 - 1) / dt, "k_sum": s.k_sum,
       "k_max_observed": s.k_max_observed,
       "histogram": {k: c for k, c in enumerate(s.histogram) if c}, "records": rec,
       "clocks": clocks.summary()}
if log2 == 50:
    paper = {1: 11, 2: 29, 3: 533, 4: 849, 5: 434977, 6: 10329791, 7: 28819433, 8: 129747557,
             9: 6915752957, 10: 2569472629649, 11: 23373845739407, 12: 60690478781437}
    out["paper_k_sum_ok"] = s.k_sum == 684465092067182
    out["paper_max_k_ok"] = s.k_max_observed == 13
    out["paper_records_ok"] = all(rec.get(m) == n for m, n in paper.items())
print(json.dumps(out, indent=1))
