"""Whole-call time of a library variant (graph replay and PDL on, as in
bench.py's `value`): python tools/exp_step.py LIB.so|- [START END] [--reps N]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--reps")]
reps = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--reps=")), "5"))
if args and args[0] != "-":
    os.environ["SQF2K_LIB"] = str(Path(args[0]).resolve())
if os.environ.get("IMPORT_TORCH"):  # torch's CUDA context first, as bench.py has it
    import torch

    torch.zeros(1, device="cuda")
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

start = int(eval(args[1])) if len(args) > 1 else (1 << 50) - (1 << 44) + 1
end = int(eval(args[2])) if len(args) > 2 else 1 << 50
end += (end - start) % 2
pipeline = os.environ.get("PIPELINE", "fused")
batch = int(eval(os.environ.get("BATCH", "0")))
for _ in range(3):
    verify_range(start, end, 30, pipeline=pipeline, batch_slots=batch)
ts = []
for _ in range(reps):
    _lib.sync()
    t = time.perf_counter()
    s = verify_range(start, end, 30, pipeline=pipeline, batch_slots=batch)
    ts.append(time.perf_counter() - t)
name = Path(args[0]).name if args and args[0] != "-" else "main"
best = min(ts)
print(f"{name:>24}: call {best * 1e3:.3f} ms (median {sorted(ts)[len(ts) // 2] * 1e3:.3f})  "
      f"{(end - start) // 2 / best / 1e12:.2f}e12 odd n/s  k_sum={s.k_sum}", flush=True)
