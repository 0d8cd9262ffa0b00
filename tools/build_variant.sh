#!/bin/bash
# Build an exploration copy of the library with extra -D flags: tools/build_variant.sh NAME -DFOO=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/.."
out=build/var_$name; mkdir -p $out
objs=""
for f in paper_2306_14316_b200/csrc/*.cu; do
  o=$out/$(basename $f .cu).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include "$@" -c $f -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libim2win_sm100.so $objs
echo $out/libim2win_sm100.so
