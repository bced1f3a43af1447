"""Per-source-line instruction counts and stall samples from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep [TOP]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "-") and r[2] == "-":
        try:
            ie = int(r[7])
            st = int(r[4])
        except ValueError:
            continue
        if ie or st:
            out.append((ie, st, cur, r[0], r[1][:100]))
tot = sum(o[0] for o in out) or 1
tst = sum(o[1] for o in out) or 1
print(f"total warp instructions {tot}, stall samples {tst}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0]:>11} {100*o[0]/tot:5.1f}%  stall {100*o[1]/tst:5.1f}%  {o[2]}:{o[3]:<5} {o[4]}")
