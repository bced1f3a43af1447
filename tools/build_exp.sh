#!/bin/bash
# build experiment variants of the library into /tmp-free in-tree names: lib_exp_<name>.so
cd "$(dirname "$0")/.."
src=paper_2411_01964_b200/csrc
for v in "$@"; do
  name=${v%%=*}; flags=${v#*=}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -shared -cudart static -diag-suppress 186 -I include $flags -o experiments/lib_exp_$name.so $src/context.cu $src/primes.cu $src/tile.cu $src/verify.cu $src/scan.cu &
done
wait
