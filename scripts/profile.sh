#!/bin/bash
# ncu evidence for bench.py (one GPU).  Each ncu command runs only after the same
# command line exited 0 without ncu.
set -u
mkdir -p gpurun_out
# 1. launch list of the bench command (device time of every launch)
CMD="python bench.py --steps 2 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch.log
# 2. full-size DRAM traffic of the momentum/score kernels (the dominant kernel of the step)
CMD1="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
$CMD1 > gpurun_out/prof_plain1.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:k_momentum_score|k_scatter_cols|k_gather_rows|k_scatter_rows|k_ns_apply" -c 8 --csv --log-file gpurun_out/k1_traffic.csv $CMD1 > gpurun_out/ncu_k1.log 2>&1
echo "k1 traffic exit $?" >> gpurun_out/ncu_k1.log
# 3. --set full of the main kernels of one step on 6 of the 24 layers
CMD2="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep --layers ${PROF_LAYERS:-6}"
$CMD2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${PROF_KERNELS:-k_ns_|k_gather_rows|k_scatter_cols|k_momentum_score|k_topk|k_scatter_rows|k_col_scores}" -s ${PROF_SKIP:-0} -c ${PROF_COUNT:-8} -o gpurun_out/prof $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full.log
