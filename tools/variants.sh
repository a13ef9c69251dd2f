#!/bin/bash
# Build libgenred variants that differ only in one source file's compile flags:
#   tools/variants.sh <src-basename> tag "-DFLAG=.." [tag2 "flags2" ...] -> build/var/libgenred_<tag>.so
set -e
cd "$(dirname "$0")/.."
src=$1; shift
python -m paper_2004_11127_b200.build >/dev/null
mkdir -p build/var
OBJS=$(ls build/genred/*.o | grep -v "/$src\.")
pids=""; tags=""
while [ $# -gt 0 ]; do
  tag=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -Iinclude $flags -c paper_2004_11127_b200/csrc/$src.cu -o build/var/${src}_$tag.o &
  pids="$pids $!"; tags="$tags $tag"
done
wait $pids
for tag in $tags; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/var/libgenred_$tag.so $OBJS build/var/${src}_$tag.o
  echo build/var/libgenred_$tag.so
done
