#!/bin/bash
# Build a variant of the C-ABI library with extra nvcc flags (profiling ablations):
#   scripts/build_variant.sh NAME -DFSP_BWD_ABLATE=2 ...   -> paper_2412_01523_b200/_lib/variants/NAME.so
# Select it at run time with FSP_LIB=paper_2412_01523_b200/_lib/variants/NAME.so
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_2412_01523_b200/_lib/variants/$name
mkdir -p "$out"
objs=()
for src in "$root"/paper_2412_01523_b200/csrc/*.cu; do
  o=$out/$(basename "${src%.cu}").o
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
    -gencode arch=compute_100a,code=sm_100a "$@" -I "$root/include" -c "$src" -o "$o" &
  objs+=("$o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out.so" "${objs[@]}" -lcuda
echo "$out.so"
