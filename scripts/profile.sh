#!/bin/bash
# ncu evidence for bench.py (one GPU).  Each ncu command runs only after the same
# command line exited 0 without ncu.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-alpha1 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch.log
CMD2="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --layers ${PROF_LAYERS:-6}"
$CMD2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${PROF_KERNELS:-k_ns_gemm_tc|k_gather_cols_t|k_scatter_cols_t|k_momentum_score_rows}" -s ${PROF_SKIP:-28} -c ${PROF_COUNT:-6} -o gpurun_out/prof $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full.log
