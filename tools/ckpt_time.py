"""C5 through run_verify with and without a checkpoint file (batch-granular
checkpoints, runner.CHECKPOINT_SPAN), wall-clock per run.

    python tools/ckpt_time.py [--reps 3]
"""

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--log2w", type=int, default=44)
    a = ap.parse_args()
    from paper_2411_01964_b200 import runner
    from paper_2411_01964_b200.aggregate import render_report_json
    from paper_2411_01964_b200.runner import RunConfig, run_verify

    start, end = (1 << 50) - (1 << a.log2w) + 1, 1 << 50
    run_verify(RunConfig(start=start, end=end))
    out = {"range": [start, end], "checkpoint_span": runner.CHECKPOINT_SPAN}
    plain, ck = [], []
    ref = None
    for _ in range(a.reps):
        t = time.perf_counter()
        rep = run_verify(RunConfig(start=start, end=end))
        plain.append(time.perf_counter() - t)
        ref = render_report_json(rep)
        with tempfile.TemporaryDirectory() as d:
            cfg = RunConfig(start=start, end=end, checkpoint_path=Path(d) / "cp.txt")
            t = time.perf_counter()
            rep2 = run_verify(cfg)
            ck.append(time.perf_counter() - t)
            assert render_report_json(rep2) == ref
            out["checkpoint_sequence"] = rep2.sequence
    out["plain_s"] = plain
    out["checkpointed_s"] = ck
    out["overhead"] = min(ck) / min(plain) - 1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
