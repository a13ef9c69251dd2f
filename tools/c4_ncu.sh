python tools/profile_run.py --what argk --M 10000 --N 60000 --D 784 --K 10 --reps 2 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rerank|split" -s 3 -c 3 -o gpurun_out/c4_aux2 python tools/profile_run.py --what argk --M 10000 --N 60000 --D 784 --K 10 --reps 2 > gpurun_out/ncu_c4aux.log 2>&1
ncu -i gpurun_out/c4_aux2.ncu-rep --page source --csv --kernel-name regex:rerank > gpurun_out/c4_rerank_source.csv 2>&1
