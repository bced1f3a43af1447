"""Benchmark of the sqf2k hot path on B200: odd n verified per second.

    python bench.py [--config C5] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1)

Workload (default "C5", BASELINE.json configs[4], the north-star range): the
2^44-wide window ending at 2^50, i.e. the reference's
`run_verify(RunConfig(start=2**50 - 2**44 + 1, end=2**50))` at its defaults
(segment width 2^30, k_max 30) -- 2^43 odd n, 2,063,689 bucketed primes.
`--config C2|C3|C4` selects the other named ranges.  Under
N GPUs the SAME range is split into N contiguous odd-aligned shards, one per
rank, reduced over NCCL (strong scaling).

A step = one pass of the hot path over the workload:
  value : device-timed (CUDA events on the library stream) sqf2k_verify of
          the rank's shard -- prime table, bucket lists, fused tile kernel,
          reduction -- max over ranks; L2 flushed between steps.
  e2e   : the public API `run_verify(RunConfig(...))` (C ABI, host buffers,
          summary/failure copies, NCCL merge, recheck, records), wall-timed,
          max over ranks; L2 flushed between steps as for `value`.
  secondary : the C2 range ([1, 1.4e9), BASELINE.json configs[1]) measured
          the same way (N = 1 only).
The CPU baseline and the reference arm (`--impl reference`) time the oracle
port (C restatement of the reference algorithm, oracle/, all host cores) on a
bounded sample of the workload: for C4/C5 the 2^34-wide sub-window ending at
2^50 (the per-n cost is flat at a fixed magnitude), whose
rate is the C4/C5 rate, "extrapolated".
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

METRIC = "odd n verified/sec (min-k per n) at 1/2/4/8 B200; fraction of roofline"
BYTES_PER_ODD_N = 0.25  # 1 bit written by the sieve + 1 bit read by the scan
K_MAX = 30
WIDTH = 1 << 30
TOP = 1 << 50

# name -> (start, end, description), BASELINE.json configs
CONFIGS = {
    "C2": (1, 1_400_000_000, "C2: verify all odd n < 1.4e9 (BASELINE.json configs[1])"),
    "C3": (1, 1 << 36, "C3: verify all odd n < 2^36 (BASELINE.json configs[2])"),
    "C4": (TOP - (1 << 40) + 1, TOP,
           "C4: 2^40-wide window ending at 2^50 (BASELINE.json configs[3])"),
    "C5": (TOP - (1 << 44) + 1, TOP,
           "C5: 2^44-wide window ending at 2^50, the north-star sweep (BASELINE.json configs[4])"),
}
# bounded CPU samples (start, end, label) of each workload
CPU_SAMPLES = {
    "C2": (1, 1_400_000_000, "the whole C2 range"),
    "C3": (1, 1 << 34, "[1, 2^34), a quarter of C3 (rate extrapolated to C3)"),
    "C4": (TOP - (1 << 34) + 1, TOP, "the 2^34-wide sub-window ending at 2^50, extrapolated x64 to C4"),
    "C5": (TOP - (1 << 34) + 1, TOP, "the 2^34-wide sub-window ending at 2^50, extrapolated x1024 to C5"),
}


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def odd_count(start: int, end: int) -> int:
    return 0 if end <= start else end // 2 - start // 2


def n_odd_scanned(start: int, end: int) -> int:
    """Odd n a run over [start, end) scans (n = 1 excluded; effective end)."""
    eff = end + 1 if (end - start) % 2 else end
    return odd_count(start, eff) - (1 if start == 1 else 0)


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
        sm, mx, power, reasons = [], 0.0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ ours -----

class _Dist:
    def __init__(self, world: int, backend: str = "nccl"):
        self.world = world
        self.device = "cuda" if backend == "nccl" else "cpu"

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self) -> None:
        import torch

        torch.cuda.synchronize()
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()


def measure(name: str, args, D: _Dist, rank: int, flush, stream, peak: float,
            peak_src: str, clocks: ClockSampler | None = None) -> dict:
    """value / e2e / per-kernel roofline of one named range on this job."""
    import torch

    from paper_2411_01964_b200 import _lib
    from paper_2411_01964_b200.runner import RunConfig, run_verify, verify_range
    from paper_2411_01964_b200.shard import shard_bounds

    start, end, desc = CONFIGS[name]
    eff_end = end + 1 if (end - start) % 2 else end
    lo, hi = shard_bounds(start, eff_end, D.world, rank)
    n_odd = n_odd_scanned(start, end)

    def step_device():
        return verify_range(lo, hi, K_MAX, pipeline=args.pipeline)

    # warm-up: at least W steps and min_warmup_s seconds (clocks settle)
    t_warm = time.perf_counter()
    done = 0
    while done < args.warmup or time.perf_counter() - t_warm < args.min_warmup_s:
        step_device()
        done += 1
    if clocks is not None:
        clocks.__enter__()
    # --- device-timed steps (value): no per-kernel events in the way -------
    times = []
    D.barrier()
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
    ms = D.max(sum(times) / len(times))
    # --- end to end through the public API (e2e) ---------------------------
    cfg = RunConfig(start=start, end=end, segment_width=WIDTH, pipeline=args.pipeline)
    run_verify(cfg)
    _lib.profile_reset()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        D.barrier()
        t0 = time.perf_counter()
        rep = run_verify(cfg)
        e2e_times.append(time.perf_counter() - t0)
    h2d, d2h = _lib.copy_stats()
    e2e_s = D.max(sum(e2e_times) / len(e2e_times))
    if clocks is not None:
        clocks.__exit__(None, None, None)
    D.barrier()
    # --- per-kernel breakdown: the same steps with every launch bracketed ---
    _lib.profile(True)
    _lib.profile_reset()
    prof_steps = max(1, min(args.steps, args.prof_steps))
    for _ in range(prof_steps):
        flush.zero_()
        torch.cuda.synchronize()
        step_device()
    kstats = _lib.profile_read()
    _lib.profile(False)

    top_name, (launches, total_ms) = max(kstats.items(), key=lambda kv: kv[1][1])
    per_launch_ms = total_ms / max(launches, 1)
    # slots of this rank's shard, spread over its tile launches (one per batch)
    units_per_launch = (hi - lo) // 2 * prof_steps / max(launches, 1)
    achieved = units_per_launch * BYTES_PER_ODD_N / (per_launch_ms / 1e3) / 1e9
    traffic = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        ent = json.loads(tj.read_text()).get(f"{top_name}@{name}")
        if ent and ent.get("pipeline") == args.pipeline:
            traffic = ent["dram_bytes_per_launch"]
    launches_per_step = sum(v[0] for v in kstats.values()) / prof_steps
    out = {
        "value": n_odd / (ms / 1e3),
        "ms_per_step": ms,
        "workload": desc,
        "range": [start, end],
        "roofline": {
            "bound": "hbm", "kernel": top_name,
            "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "algorithmic_bytes_per_odd_n": BYTES_PER_ODD_N,
            "odd_n_per_launch": units_per_launch,
            "kernel_ms_per_launch": per_launch_ms,
            "kernel_share_of_step": (total_ms / prof_steps) / (sum(times) / len(times)),
            "how": "per-launch CUDA events on the launching stream (profile mode: PDL, graph "
                   "replay and the side-stream overlap of multi-batch calls off, so each "
                   "kernel is timed alone) over extra steps of the same call",
        },
        "kernels": {k: {"launches_per_step": v[0] / prof_steps, "ms_per_step": v[1] / prof_steps}
                    for k, v in sorted(kstats.items())},
        "launches_per_step": launches_per_step,
        "e2e": {"value": n_odd / e2e_s, "unit": "odd n/s", "s_per_step": e2e_s,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "api": "paper_2411_01964_b200.run_verify(RunConfig(...))",
                "k_sum": rep.summary.k_sum, "k_max_observed": rep.summary.k_max_observed},
        "warmup_steps_run": done,
    }
    pin = _pinned_k_sum(name)
    if pin is not None:
        out["e2e"]["k_sum_pinned"] = pin
        if rep.summary.k_sum != pin:
            raise SystemExit(f"{name}: k_sum {rep.summary.k_sum} != reference {pin}")
    return out


def _pinned_k_sum(name: str) -> int | None:
    """k_sum of the reference's own report for this range (tests/golden)."""
    start, end, _ = CONFIGS[name]
    g = ROOT / "tests" / "golden"
    for f in ("golden_large.json", "golden_window_2p40.json", "golden_window_2p44.json"):
        p = g / f
        if not p.exists():
            continue
        d = json.loads(p.read_text())
        for e in d.get("verify", [d]):
            c = e.get("config", {})
            if c.get("start") == start and c.get("end") == end:
                return int(e["summary"]["k_sum"])
    return None


def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    # SQF2K_BENCH_BACKEND=gloo + SQF2K_DEVICE: the N > 1 code path with every
    # rank on one GPU (tests/test_gpu_multirank.py); the product runs NCCL
    backend = os.environ.get("SQF2K_BENCH_BACKEND", "nccl")
    device = int(os.environ.get("SQF2K_DEVICE", local))
    torch.cuda.set_device(device)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)

    from paper_2411_01964_b200 import _lib

    _lib.lib()  # bind this rank's GPU; raises without the native library
    D = _Dist(world, backend)
    stream = torch.cuda.ExternalStream(_lib.stream_handle())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    peak, peak_src = measured_peak_gbs()

    clocks = ClockSampler(device)
    head = measure(args.config, args, D, rank, flush, stream, peak, peak_src, clocks)
    secondary = None
    if world == 1 and args.config != "C2" and not args.no_secondary:
        secondary = measure("C2", args, D, rank, flush, stream, peak, peak_src)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return None

    start, end = head["range"]
    line = {
        "metric": METRIC,
        "value": head["value"],
        "unit": "odd n/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32/u64 (bit-packed integer)",
        "data": "the integer range itself (deterministic, no dataset)",
        "config": {
            "workload": head["workload"] + (f", range-sharded over {world} GPUs" if world > 1 else ""),
            "range": [start, end], "k_max": K_MAX, "segment_width": WIDTH,
            "pipeline": args.pipeline, "parallelism": f"range-sharded x{world}",
            "l2": "flushed between timed steps (256 MiB write)",
        },
        "roofline": head["roofline"],
        "kernels": head["kernels"],
        "gpu_launches": int(round(head["launches_per_step"] * args.steps)),
        "e2e": head["e2e"],
        "clocks": clocks.summary(),
        "warmup_steps_run": head["warmup_steps_run"],
    }
    if secondary is not None:
        line["secondary"] = {k: secondary[k] for k in
                             ("workload", "range", "value", "ms_per_step", "roofline", "kernels", "e2e")}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    return line


# -------------------------------------------------------- CPU reference ------

def cpu_baseline(name: str, threads: int | None = None) -> dict:
    """The oracle port (C restatement of the reference's segment loop,
    oracle/) on the host cores, on the config's bounded sample at the
    reference defaults (W = 2^30, k_max 30)."""
    from oracle import oracle as O

    threads = threads or os.cpu_count() or 1
    O.build()
    s, e, label = CPU_SAMPLES[name]
    t0 = time.perf_counter()
    res = O.verify(s, e + 1 if (e - s) % 2 else e, width=WIDTH, k_max=K_MAX, threads=threads)
    dt = time.perf_counter() - t0
    n = n_odd_scanned(s, e)
    rate = n / dt
    whole = n_odd_scanned(*CONFIGS[name][:2])
    return {"value": rate, "unit": "odd n/s", "cores": threads, "kind": "port",
            "sample": f"{label}: [{s}, {e}) = {n} odd n in {dt:.2f} s",
            "extrapolated": whole != n,
            "workload_seconds": whole / rate, "k_sum": res["k_sum"]}


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    from oracle import oracle as O

    O.build()
    s, e, _ = CPU_SAMPLES[args.config]
    ws = max(s, (e - (1 << 26)) | 1)  # short warm-up windows at the same magnitude
    for _ in range(args.warmup):
        O.verify(ws, e + 1 if (e - ws) % 2 else e, width=WIDTH, k_max=K_MAX,
                 threads=os.cpu_count() or 1)
    vals = []
    b = None
    for _ in range(args.steps):
        b = cpu_baseline(args.config)
        vals.append(b["value"])
    v = statistics.median(vals)
    start, end, desc = CONFIGS[args.config]
    n = n_odd_scanned(s, e)
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "odd n/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n / v, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "the integer range itself",
        "config": {"workload": desc, "range": [start, end], "k_max": K_MAX,
                   "segment_width": WIDTH, "sample_range": [s, e]},
        "cpu_baseline": {"value": v, "unit": "odd n/s", "cores": b["cores"], "kind": "port",
                         "sample": b["sample"], "extrapolated": b["extrapolated"]},
        "e2e": {"value": v, "unit": "odd n/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C5")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pipeline", choices=["fused", "bitmap"], default="fused")
    ap.add_argument("--prof-steps", type=int, default=3,
                    help="steps re-run with per-launch events for the kernel breakdown")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C2 secondary line")
    ap.add_argument("--min-warmup-s", type=float, default=1.5,
                    help="keep warming up at least this long (clocks settle)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
