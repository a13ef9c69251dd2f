python tools/profile_run.py --what argk --M 10000 --N 60000 --D 784 --K 10 --reps 3 > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/profile_run.py --what argk --M 10000 --N 60000 --D 784 --K 10 --reps 3 > gpurun_out/ncu_c4.log 2>&1
