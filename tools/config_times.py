"""Wall time of run_verify on the BASELINE.json configs C3..C5 (one GPU)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import RunConfig, run_verify  # noqa: E402

cfgs = {"C3": (1, 1 << 36), "C4": ((1 << 50) - (1 << 40) + 1, 1 << 50),
        "C5": ((1 << 50) - (1 << 44) + 1, 1 << 50)}
out = {}
for name, (s, e) in cfgs.items():
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    cfg = RunConfig(start=s, end=e)
    run_verify(cfg)  # warm-up: buffers, the call's CUDA graph
    _lib.sync()
    t = time.perf_counter()
    rep = run_verify(cfg)
    dt = time.perf_counter() - t
    n = rep.summary.odd_scanned
    out[name] = {"range": [s, e], "seconds": dt, "odd_n_per_s": n / dt, "k_sum": rep.summary.k_sum,
                 "k_max_observed": rep.summary.k_max_observed}
    print(name, json.dumps(out[name]), flush=True)
