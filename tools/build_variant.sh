#!/bin/bash
# Build a variant of libspecdec_b200.so with extra nvcc flags (A/B timing on
# the GPU box via SDB_LIB=...).  usage: tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
name=$1; shift
flags="$*"
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2508_08192_b200/csrc
out=$root/tools/variants/$name
mkdir -p "$out/obj"
for f in "$src"/*.cu; do
  b=$(basename "$f" .cu)
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
    --expt-relaxed-constexpr $flags -Xptxas -v -c "$f" -o "$out/obj/$b.o" 2> "$out/obj/$b.ptxas.txt" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libspecdec_b200.so" "$out"/obj/*.o -lcuda
echo "$out/libspecdec_b200.so"
