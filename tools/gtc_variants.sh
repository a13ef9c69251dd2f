#!/bin/bash
# Build libgenred variants differing only in gauss_tc.cu compile flags:
#   tools/gtc_variants.sh tag "-DFLAG=.. -DFLAG2=.." [tag2 "flags2" ...]  -> build/gtcv/libgenred_<tag>.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2004_11127_b200.build >/dev/null
mkdir -p build/gtcv
OBJS=$(ls build/genred/*.o | grep -v "/gauss_tc\.")
while [ $# -gt 0 ]; do
  tag=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -Iinclude $flags -c paper_2004_11127_b200/csrc/gauss_tc.cu -o build/gtcv/gtc_$tag.o &
  pids="$pids $!"; tags="$tags $tag"
done
wait $pids
for tag in $tags; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/gtcv/libgenred_$tag.so $OBJS build/gtcv/gtc_$tag.o
  echo build/gtcv/libgenred_$tag.so
done
