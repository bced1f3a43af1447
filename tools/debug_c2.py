import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O
from paper_2411_01964_b200.primes import generate_primes
from paper_2411_01964_b200.runner import verify_range
from paper_2411_01964_b200.sieve import sieve_segment

end = 1400000001
for pipe in ("bitmap", "fused"):
    for depth in (0, 14, 12):
        print(pipe, depth, verify_range(1, end, 30, pipeline=pipe, tile_depth=depth).k_sum, flush=True)
# export bitmap vs oracle on [1, 2^28)
e2 = (1 << 28) + 1
p = generate_primes(int(np.sqrt(e2)) + 2)
g = sieve_segment(1, e2, p).bits
o = O.sieve_bits(1, e2, p.primes, p.limit)
d = np.flatnonzero(g != o)
print("export mismatched bytes", len(d), d[:10])
# fused on pieces
for lo, hi in [(1, 1 << 25), (1 << 25, 1 << 26), (1 << 26, 1 << 27), (1, 1 << 27)]:
    lo |= 1; hi |= 1
    want = O.verify(lo, hi, width=1 << 30, k_max=30)["k_sum"]
    got = verify_range(lo, hi, 30).k_sum
    print("fused", lo, hi, got, want, got == want, flush=True)
