"""Small driver for ncu captures: verify_range over a range a few times.

    python tools/prof_verify.py START END [--k-max 30] [--pipeline fused] [--reps 3]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01964_b200.runner import verify_range  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("start", type=lambda s: int(eval(s)))
ap.add_argument("end", type=lambda s: int(eval(s)))
ap.add_argument("--k-max", type=int, default=30)
ap.add_argument("--pipeline", default="fused")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--batch", type=lambda s: int(eval(s)), default=0)
a = ap.parse_args()
end = a.end + ((a.end - a.start) % 2)
for i in range(a.reps):
    t = time.perf_counter()
    s = verify_range(a.start, end, a.k_max, pipeline=a.pipeline, batch_slots=a.batch)
    print(f"rep {i}: {time.perf_counter() - t:.4f}s k_sum={s.k_sum} kmo={s.k_max_observed}", flush=True)
