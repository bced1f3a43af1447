# Random search over the medium-schedule constants (SQF2K_MED_*, read by
# build_med) on the C5 window: bash tools/sched_search.sh (on the GPU box)
cd "$(dirname "$0")/.."
python - <<'PY'
import random, subprocess, os, re
rng = random.Random(5)
cands = [(7.5, 0.25, 2.0, 2.0)]
for _ in range(40):
    cands.append((round(rng.uniform(5.5, 9.5), 2), rng.choice([0.0, 0.25, 0.5, 0.75, 1.0]),
                  rng.choice([1.5, 2.0, 2.5, 3.0]), rng.choice([0.0, 1.0, 2.0, 4.0])))
res = []
for it, b, pt, tk in cands:
    env = dict(os.environ, SQF2K_MED_ITEM=str(it), SQF2K_MED_BIAS=str(b), SQF2K_MED_PER_TRIP=str(pt), SQF2K_MED_TASK=str(tk))
    out = subprocess.run(["python", "tools/exp_step.py", "-", "--reps=3"], env=env, capture_output=True, text=True).stdout
    m = re.search(r"call ([0-9.]+) ms", out)
    t = float(m.group(1)) if m else 1e9
    res.append((t, it, b, pt, tk))
    print(f"{t:.3f} item {it} bias {b} per_trip {pt} task {tk}", flush=True)
res.sort()
print("BEST", res[:5])
PY
