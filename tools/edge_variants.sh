# HBM-bound edge kernel (M = 2^28, N = 1 and 8) across library variants (VARS or build/var/*.so).
for lib in ${VARS:-build/var/libgenred_*.so}; do
  for n in 1 8; do
    echo -n "lib $lib N $n "
    GENRED_LIB=$lib python bench.py --config 6 --edge-n $n --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],3))"
  done
done
