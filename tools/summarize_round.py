"""Turn a tools/profile_round.sh run (gpurun_out/) into committed profiles/.

    python tools/summarize_round.py r2
"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
O, P = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"


def sh(*cmd) -> str:
    return subprocess.run(cmd, capture_output=True, text=True).stdout


for name in ["bench_c5", "bench_ref", "bench_C3", "bench_C4", "full_2p50"]:
    src = O / f"{tag}_{name}.json"
    if src.exists() and src.stat().st_size:
        shutil.copy(src, P / f"{tag}_{name}.json")

# launch list: per kernel count / mean / total, share of the captured device time
lst = O / f"{tag}_launches_c5.csv"
if lst.exists():
    rows = list(csv.reader(open(lst)))
    hdr, per = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
                per.setdefault(d["Kernel Name"].split("(")[0][-60:], []).append(us)
    tot = sum(sum(v) for v in per.values()) or 1.0
    with open(P / f"{tag}_launches_c5.txt", "w") as f:
        f.write(f"ncu --metrics gpu__time_duration.sum --clock-control none -c 800 of `python bench.py "
                f"--steps 1 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-secondary --prof-steps 1` "
                f"(C5, cold-cache serialised launches: compare shares)\n")
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k:62s} n={len(v):4d} mean={sum(v) / len(v):10.2f} us  total={sum(v) / 1e3:9.3f} ms  "
                    f"share={sum(v) / tot:6.3f}\n")
    shutil.copy(lst, P / f"{tag}_launches_c5.csv")

traffic_path = P / "ncu_traffic.json"
traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
# (the tile capture is one 2^37-slot C5 batch; the scan capture is the 2^37
# window's 2^36 slots)
for rep, out, key, algo, scale in [(f"{tag}_prof_tile_c5", f"{tag}_ncu_tile_fused_c5.txt", "tile_fused@C5", 2 ** 37 * 0.25, 1.0),
                                   (f"{tag}_prof_wscan", f"{tag}_ncu_window_scan.txt", "window_scan@2p37", 2 ** 36 / 8, 1.0)]:
    r = O / f"{rep}.ncu-rep"
    if not r.exists():
        continue
    summ = sh(sys.executable, str(ROOT / "tools/ncu_summary.py"), str(r))
    lines = sh(sys.executable, str(ROOT / "tools/ncu_lines.py"), str(r), "40")
    (P / out).write_text(summ + "\n" + lines)
    raw = sh("ncu", "-i", str(r), "--page", "raw", "--csv")
    rows = list(csv.reader(raw.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))

    def b(k):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)
        return float(d[k].replace(",", "")) * scale
    traffic[key] = {"pipeline": "fused" if "tile" in key else "bitmap",
                    "dram_bytes_per_launch": scale * (b("dram__bytes_read.sum") + b("dram__bytes_write.sum")),
                    "algorithmic_bytes_per_launch": algo,
                    "source": f"profiles/{out} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum"
                              + (f", x{scale:g} from a smaller launch)" if scale != 1.0 else ")")}
traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
print("profiles written")
