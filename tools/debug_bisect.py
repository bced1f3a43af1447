import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O
from paper_2411_01964_b200.runner import verify_range

def bad(lo, hi, depth):
    want = O.verify(lo, hi, width=1 << 30, k_max=30)
    got = verify_range(lo, hi, 30, tile_depth=depth)
    return got.histogram != want["histogram"], got, want

for ntiles in range(1, 8):
    hi = 1 + 2 * ntiles * 32768
    b, g, w = bad(1, hi, 10)
    print("tiles", ntiles, "bad", b, flush=True)
# bisect on hi within 6 tiles
lo_hi, hi_hi = 1 + 2 * 5 * 32768, 1 + 2 * 6 * 32768
if bad(1, hi_hi, 10)[0]:
    a, b_ = lo_hi, hi_hi
    print("prefix 5 tiles bad:", bad(1, a, 10)[0])
    while b_ - a > 2:
        m = (a + b_) // 2
        m -= (m - 1) % 2
        if bad(1, m, 10)[0]:
            b_ = m
        else:
            a = m
    print("first bad end", b_, "n =", b_ - 2)
    _, g, w = bad(1, b_, 10)
    print([(k, g.histogram[k], w["histogram"][k]) for k in range(20) if g.histogram[k] != w["histogram"][k]])
