"""Per-source-line stall reasons from an ncu report (source page, CUDA view).

    python tools/ncu_stalls.py REPORT.ncu-rep [TOP]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur, hdr, out, tot = None, None, [], {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        d = dict(zip(hdr, r))
        d["Source"] = r[1]
        st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
        n = sum(st.values())
        if n:
            out.append((n, f"{cur}:{d['Line No']}", d["Source"][:60], st))
            for k, v in st.items():
                tot[k] = tot.get(k, 0) + v
T = sum(tot.values()) or 1
print("all samples by reason:", ", ".join(f"{k} {v / T:.1%}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
for n, where, src, st in sorted(out, reverse=True)[:top]:
    top3 = ", ".join(f"{k} {v / n:.0%}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4] if v)
    print(f"{n / T:6.1%}  {where:<18} {src:<60} | {top3}")
