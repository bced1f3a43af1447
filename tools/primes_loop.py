import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib
L = _lib.lib()
c = ctypes.c_uint64(0)
for i in range(40):
    L.sqf2k_prime_count(37416 - 2 * i, ctypes.byref(c))
print(c.value)
