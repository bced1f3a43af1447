"""Per-CTA timeline of the tile kernel (experiment build with -DSQF2K_EXP_TIMELINE):
python tools/timeline.py LIB.so START END"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2411_01964_b200 import _lib  # noqa: E402

_lib.LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

lo, hi = int(eval(sys.argv[2])), int(eval(sys.argv[3]))
hi += (hi - lo) % 2
for _ in range(5):
    verify_range(lo, hi, 30)
L = _lib.lib()
buf = np.zeros((4096, 4), np.uint64)
L.sqf2k_exp_timeline(buf.ctypes.data_as(ctypes.c_void_p))
g = int((buf[:, 0] > 0).sum())
smid = (buf[:g, 0] >> np.uint64(56)).astype(np.int64)
buf[:g, 0] &= np.uint64((1 << 56) - 1)
b = buf[:g].astype(np.int64)
t0 = b[:, 0].min()
b = b - t0
print(f"ctas {g}: start  min {b[:,0].min()/1e3:.1f} max {b[:,0].max()/1e3:.1f} us")
print(f"prologue (start->wait) mean {np.mean(b[:,1]-b[:,0])/1e3:.1f} max {np.max(b[:,1]-b[:,0])/1e3:.1f}")
print(f"loop (wait->end) mean {np.mean(b[:,2]-b[:,1])/1e3:.1f} min {np.min(b[:,2]-b[:,1])/1e3:.1f} max {np.max(b[:,2]-b[:,1])/1e3:.1f}")
print(f"epilogue mean {np.mean(b[:,3]-b[:,2])/1e3:.1f} max {np.max(b[:,3]-b[:,2])/1e3:.1f}")
print(f"end: min {b[:,3].min()/1e3:.1f} median {np.median(b[:,3])/1e3:.1f} max {b[:,3].max()/1e3:.1f} us")
loop = (b[:, 2] - b[:, 1]) / 1e3
dec = np.array_split(np.arange(g), 16)
print("loop us by CTA index (16 groups):", " ".join(f"{loop[d].mean():.1f}" for d in dec))
print("end us by CTA index (16 groups):", " ".join(f"{b[d, 3].mean() / 1e3:.1f}" for d in dec))
sm = np.arange(g) % 148
if g == 592:
    per_sm = loop.reshape(4, 148)  # CTA b and b + 148k share an SM if dispatch is round-robin
    print("per-SM mean spread: min %.1f max %.1f; within-SM spread mean %.1f" % (
        per_sm.mean(0).min(), per_sm.mean(0).max(), (per_sm.max(0) - per_sm.min(0)).mean()))
    print("corr of CTA b with b+148:", np.corrcoef(per_sm[0], per_sm[1])[0, 1])
loop_by_sm = np.zeros(200); cnt = np.zeros(200)
np.add.at(loop_by_sm, smid, loop); np.add.at(cnt, smid, 1)
m = loop_by_sm[cnt > 0] / cnt[cnt > 0]
ids = np.nonzero(cnt > 0)[0]
order = np.argsort(m)
print("slowest SMs:", [(int(ids[i]), round(float(m[i]))) for i in order[-12:]])
print("fastest SMs:", [(int(ids[i]), round(float(m[i]))) for i in order[:12]])
np.save("gpurun_out/sm_loop.npy", np.stack([ids, m]))
if g == 592:
    waves = loop.reshape(4, 148)
    print("loop by wave (blockIdx // 148): mean", [round(float(x), 1) for x in waves.mean(1)],
          "min", [round(float(x), 1) for x in waves.min(1)], "max", [round(float(x), 1) for x in waves.max(1)])
    sm_of = smid.reshape(4, 148)
    print("same SM for b and b+148?", float((sm_of[0] == sm_of[1]).mean()), "smid of 0..7:", smid[:8].tolist(), "148..155:", smid[148:156].tolist())
# within-SM rank by start time vs loop time
ranks = {}
for i in range(g):
    ranks.setdefault(int(smid[i]), []).append(i)
by_rank = [[], [], [], [], [], []]
by_bidx = [[], [], [], [], [], []]
for sm, ids in ranks.items():
    if len(ids) > 6 or len(ids) < 1:
        continue
    order = sorted(ids, key=lambda i: b[i, 0])
    for r, i in enumerate(order):
        by_rank[r].append(loop[i])
    for r, i in enumerate(sorted(ids)):
        by_bidx[r].append(loop[i])
print("group sizes", sorted(set(len(v) for v in ranks.values())))
print("loop by start-rank on SM:", [round(float(np.mean(x)), 1) for x in by_rank if x])
print("loop by blockIdx-rank on SM:", [round(float(np.mean(x)), 1) for x in by_bidx if x])
print("loop by blockIdx % 4:", [round(float(loop[np.arange(g) % 4 == j].mean()), 1) for j in range(4)])
print("loop by blockIdx % 4 (std):", [round(float(loop[np.arange(g) % 4 == j].std()), 1) for j in range(4)])
