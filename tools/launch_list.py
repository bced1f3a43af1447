"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel count, mean, min (us)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) / (1000.0 if d.get("Metric Unit") in ("ns", "nsecond") else 1.0)
            out.setdefault(d["Kernel Name"][:70], []).append(v)
for k, v in out.items():
    print(f"{k:70s} n={len(v):4d} mean={sum(v) / len(v):9.2f} us  min={min(v):9.2f} us")
