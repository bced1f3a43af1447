"""Group per-line instruction counts of an ncu report into categories given
as FILE:LO-HI ranges.   python tools/ncu_cats.py REP name=file:lo-hi ..."""
import csv
import subprocess
import sys

rep = sys.argv[1]
cats = []
for a in sys.argv[2:]:
    name, spec = a.split("=")
    f, rng = spec.split(":")
    lo, hi = map(int, rng.split("-"))
    cats.append((name, f, lo, hi))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur, hdr = None, None
tot = {c[0]: [0, 0] for c in cats}
tot["other"] = [0, 0]
allsum = [0, 0]
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "-") and r[2] == "-":
        try:
            ie, st = int(r[7]), int(r[4])
        except ValueError:
            continue
        ln = int(r[0])
        key = "other"
        for name, f, lo, hi in cats:
            if cur == f and lo <= ln <= hi:
                key = name
                break
        tot[key][0] += ie
        tot[key][1] += st
        allsum[0] += ie
        allsum[1] += st
for k, (ie, st) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:>12} {ie:>11} {100*ie/allsum[0]:5.1f}%  stall {100*st/allsum[1]:5.1f}%")
