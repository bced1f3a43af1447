"""Random large windows (widths 2^30..2^44 at magnitudes 2^36..2^62), this library vs another
build (default: round 1's, experiments/lib_exp_r1.so): histogram, k_sum, records, failures.
    WIDTHS="[41, 44]" NCASES=8 python tools/stress_vs_build.py [LIB] [SEED]"""
import os, random, subprocess, sys, json
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
other = sys.argv[1] if len(sys.argv) > 1 else "experiments/lib_exp_r1.so"
WIDTHS = json.loads(os.environ.get("WIDTHS", "[30, 33, 35, 37, 38, 39, 40]"))
NCASES = int(os.environ.get("NCASES", "24"))
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
cases = []
for _ in range(NCASES):
    mag = rng.choice([36, 40, 44, 48, 52, 56, 60, 62])
    width = 1 << rng.choice(WIDTHS)
    end = min(1 << mag, (1 << 62) - 1)
    start = max(1, end - width - rng.randrange(0, 1 << 20))
    start |= 1
    end = start + 2 * ((end - start) // 2)
    batch = rng.choice([0, 0, 1 << 34, (1 << 33) + (1 << 16) * 3])
    cases.append((start, end, batch))
code = r'''
import json, sys
sys.path.insert(0, ROOT)
from paper_2411_01964_b200.runner import verify_range
out = []
for s, e, b in CASES:
    r = verify_range(s, e, 30, batch_slots=b)
    out.append([r.histogram, r.k_sum, sorted(r.record_candidates.items()), r.failures])
print(json.dumps(out))
'''.replace("ROOT", repr(root)).replace("CASES", repr(cases))
res = []
for lib in (None, other):
    env = dict(os.environ)
    if lib: env["SQF2K_LIB"] = os.path.join(root, lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if r.returncode: print(lib, "FAILED", r.stderr[-800:]); sys.exit(1)
    res.append(json.loads(r.stdout.strip().splitlines()[-1]))
bad = [c for c, a, b in zip(cases, res[0], res[1]) if a != b]
print(f"{len(cases)} windows, {len(bad)} mismatches", bad[:5])
