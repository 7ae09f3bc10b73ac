#!/bin/bash
# Build measurement variants of the library into paper_2605_08523_b200/lib/var/<name>.so
#   scripts/build_variants.sh name1:"-DFLAG ..." name2:"..."
cd "$(dirname "$0")/.."
mkdir -p paper_2605_08523_b200/lib/var
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a $flags -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Iinclude -Ipaper_2605_08523_b200/csrc --expt-relaxed-constexpr -shared \
    -o paper_2605_08523_b200/lib/var/$name.so paper_2605_08523_b200/csrc/ffg_capi.cu &
done
wait
ls -la paper_2605_08523_b200/lib/var
