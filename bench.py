"""Benchmark of the sqf2k hot path on B200: odd n verified per second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1)

Workload (BASELINE.json configs[1], "C2"): verify every odd n < 1.4e9 --
the minimal exponent k of n - 2^k squarefree, histogram, k_sum, records --
i.e. reference `run_verify(RunConfig(start=1, end=1_400_000_000))` at its
defaults (segment width 2^30, k_max 30).  Under N GPUs the job is weak-scaled:
[1, N * 1.4e9) split into N contiguous shards, one per rank, reduced over NCCL.

A step = one pass of the hot path over the workload:
  value : device-timed (CUDA events on the library stream) sqf2k_verify of the
          rank's shard -- prime table, bucket lists, fused tile kernel,
          reduction -- max over ranks; L2 flushed between steps.
  e2e   : the public API `run_verify(RunConfig(...))` (C ABI, host buffers,
          summary/failure copies, NCCL merge, recheck, records) wall-timed.
The reference arm (`--impl reference`) times the oracle port (C restatement
of the reference algorithm, oracle/) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

C2_END = 1_400_000_000
METRIC = "odd n verified/sec (min-k per n) at 1/2/4/8 B200; fraction of roofline"
BYTES_PER_ODD_N = 0.25  # 1 bit written by the sieve + 1 bit read by the scan
K_MAX = 30
WIDTH = 1 << 30


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def odd_count(start: int, end: int) -> int:
    return 0 if end <= start else end // 2 - start // 2


def job_range(n_gpus: int) -> tuple[int, int]:
    return 1, 1 + n_gpus * (C2_END - 1) if n_gpus > 1 else C2_END


# ---------------------------------------------------------------- clocks -----

class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ ours -----

def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2411_01964_b200 import _lib
    from paper_2411_01964_b200.runner import RunConfig, run_verify, verify_range
    from paper_2411_01964_b200.shard import shard_bounds

    _lib.lib()  # bind this rank's GPU; raises without the native library
    start, end = job_range(world)
    lo, hi = shard_bounds(start, end, world, rank)
    stream = torch.cuda.ExternalStream(_lib.stream_handle())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def step_device():
        return verify_range(lo, hi, K_MAX, pipeline=args.pipeline)

    # clocks are sampled from the start of the warm-up to the end of the timed
    # steps (nvidia-smi samples every 100 ms; the timed steps alone are short)
    clocks = ClockSampler(local).__enter__()
    t_warm = time.perf_counter()
    done = 0
    while done < args.warmup or time.perf_counter() - t_warm < args.min_warmup_s:
        step_device()
        done += 1
    # --- device-timed steps (value): no per-kernel events in the way --------
    times = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        part = step_device()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks.__exit__(None, None, None)
    barrier()
    # --- per-kernel breakdown: the same steps with every launch bracketed ---
    _lib.profile(True)
    _lib.profile_reset()
    prof_steps = max(3, min(args.steps, 10))
    for _ in range(prof_steps):
        flush.zero_()
        torch.cuda.synchronize()
        step_device()
    kstats = _lib.profile_read()
    _lib.profile(False)
    my_ms = sum(times) / len(times)
    t = torch.tensor([my_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    n_odd = odd_count(start, end) - (1 if start == 1 else 0)
    value = n_odd / (ms / 1e3)

    # --- end to end through the public API (e2e) ---------------------------
    cfg = RunConfig(start=start, end=end, segment_width=WIDTH, pipeline=args.pipeline)
    for _ in range(max(1, args.warmup // 2)):
        run_verify(cfg)
    _lib.profile_reset()
    barrier()
    e2e_times = []
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        rep = run_verify(cfg)
        e2e_times.append(time.perf_counter() - t0)
    h2d, d2h = _lib.copy_stats()
    t = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return None

    # roofline of the dominant kernel (tile_fused, or the sieve/scan pair)
    peak, peak_src = measured_peak_gbs()
    top = max(kstats.items(), key=lambda kv: kv[1][1])
    name, (launches, total_ms) = top
    per_launch_ms = total_ms / max(launches, 1)
    # one tile launch per batch; C2 is one batch per step
    units_per_launch = (hi - lo) // 2 * prof_steps / max(launches, 1)
    achieved = units_per_launch * BYTES_PER_ODD_N / (per_launch_ms / 1e3) / 1e9
    traffic = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        ent = json.loads(tj.read_text()).get(f"{name}@C2")
        if ent and ent.get("pipeline") == args.pipeline:
            traffic = ent["dram_bytes_per_launch"]
    launches_per_step = sum(v[0] for v in kstats.values()) / prof_steps

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "odd n/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32/u64 (bit-packed integer)",
        "data": "the integer range itself (deterministic, no dataset)",
        "config": {
            "workload": "C2: verify all odd n < 1.4e9 (BASELINE.json configs[1]); "
                        f"weak-scaled to [1, {end}) over {world} GPU(s)",
            "range": [start, end], "k_max": K_MAX, "segment_width": WIDTH,
            "pipeline": args.pipeline, "parallelism": f"range-sharded x{world}",
            "l2": "flushed between timed steps (256 MiB write)",
        },
        "roofline": {
            "bound": "hbm", "kernel": name,
            "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "algorithmic_bytes_per_odd_n": BYTES_PER_ODD_N,
            "kernel_ms_per_launch": per_launch_ms,
            "kernel_share_of_step": (total_ms / prof_steps) / my_ms,
        },
        "kernels": {k: {"launches_per_step": v[0] / prof_steps, "ms_per_step": v[1] / prof_steps}
                    for k, v in sorted(kstats.items())},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "e2e": {"value": n_odd / e2e_s, "unit": "odd n/s", "s_per_step": e2e_s,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "api": "paper_2411_01964_b200.run_verify(RunConfig(...))",
                "k_sum": rep.summary.k_sum},
        "clocks": clocks.summary(),
        "warmup_steps_run": done,
    }
    if world == 1 and not args.no_large:
        line["large_window"] = large_window(peak)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(sample_end=args.cpu_sample_end)
    return line


def large_window(peak: float, log2_width: int = 37) -> dict:
    """Sustained per-kernel throughput on a 2^log2_width-integer window ending
    at 2^50 (the C4/C5 regime: 2M bucketed primes), both pipelines:
    fused tile kernel (odd n/s and the 0.25 B/n HBM-equivalent) and the
    two-pass bitmap pipeline's export (HBM write) and scan (HBM read)."""
    from paper_2411_01964_b200 import _lib
    from paper_2411_01964_b200.runner import verify_range

    end = (1 << 50) + 1
    start = end - (1 << log2_width)
    n = (end - start) // 2
    out = {"window": [start, end], "odd_n": n}
    for pipeline in ("fused", "bitmap"):
        verify_range(start, end, K_MAX, pipeline=pipeline)
        _lib.profile(True)
        _lib.profile_reset()
        reps = 3
        for _ in range(reps):
            verify_range(start, end, K_MAX, pipeline=pipeline)
        st = _lib.profile_read()
        _lib.profile(False)
        total = sum(v[1] for v in st.values()) / reps
        res = {"step_kernel_ms": total, "odd_n_per_s": n / (total / 1e3)}
        for name, (launches, ms) in st.items():
            per = ms / reps
            ent = {"ms_per_step": per, "launches_per_step": launches / reps}
            if name == "tile_fused":
                gbs = n * BYTES_PER_ODD_N / (per / 1e3) / 1e9
                ent.update(odd_n_per_s=n / (per / 1e3), hbm_equiv_gbs=gbs, frac=gbs / peak)
            if name == "tile_export":
                gbs = n / 8 / (per / 1e3) / 1e9  # one bit per odd n written
                ent.update(write_gbs=gbs, frac=gbs / peak)
            if name == "window_scan":
                gbs = n / 8 / (per / 1e3) / 1e9  # one bit per odd n read
                ent.update(read_gbs=gbs, frac=gbs / peak)
            res[name] = ent
        out[pipeline] = res
    return out


# -------------------------------------------------------- CPU reference ------

def cpu_baseline(sample_end: int, threads: int | None = None) -> dict:
    """The oracle port (C restatement of the reference's segment loop) on the
    host cores, on [1, sample_end) at the reference defaults."""
    from oracle import oracle as O

    threads = threads or os.cpu_count() or 1
    O.build()
    t0 = time.perf_counter()
    s = O.verify(1, sample_end, width=WIDTH, k_max=K_MAX, threads=threads)
    dt = time.perf_counter() - t0
    n = odd_count(1, sample_end) - 1
    return {"value": n / dt, "unit": "odd n/s", "cores": threads, "kind": "port",
            "sample": f"[1, {sample_end}) = {n} odd n, W=2^30, k_max=30, {dt:.2f} s",
            "k_sum": s["k_sum"]}


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    start, end = job_range(world)
    sample_end = min(end, args.cpu_sample_end)
    for _ in range(args.warmup):
        cpu_baseline(sample_end=min(sample_end, 1 << 24))
    vals, secs = [], []
    for _ in range(args.steps):
        b = cpu_baseline(sample_end=sample_end)
        vals.append(b["value"])
        secs.append((odd_count(1, sample_end) - 1) / b["value"])
    v = statistics.median(vals)
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "odd n/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "the integer range itself",
        "config": {"workload": "C2: verify all odd n < 1.4e9 (BASELINE.json configs[1])",
                   "range": [start, end], "k_max": K_MAX, "segment_width": WIDTH,
                   "sample_range": [1, sample_end]},
        "cpu_baseline": {"value": v, "unit": "odd n/s", "cores": b["cores"], "kind": "port",
                         "sample": b["sample"]},
        "e2e": {"value": v, "unit": "odd n/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pipeline", choices=["fused", "bitmap"], default="fused")
    ap.add_argument("--cpu-sample-end", type=int, default=C2_END)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--min-warmup-s", type=float, default=1.5,
                    help="keep warming up (and sampling clocks) at least this long")
    ap.add_argument("--no-large", action="store_true",
                    help="skip the 2^37-wide window near 2^50 per-kernel measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
