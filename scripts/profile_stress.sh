#!/bin/bash
# configs[4] (stress shapes, alpha 1/16) on one GPU: bench line, launch list, and --set full of
# the split-K gram, its reduce, and the HBM-bound gather / K1 / scatter kernels.
set -u
mkdir -p gpurun_out
CMD="python bench.py --config stress --alpha 0.0625 --steps 2 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
timeout 300 python bench.py --config stress --alpha 0.0625 --steps 10 --warmup 3 --no-e2e --no-sweep > gpurun_out/stress_bench.log 2>&1
$CMD > gpurun_out/stress_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stress_launches.csv $CMD > gpurun_out/stress_ncu_launch.log 2>&1
CMD1="python bench.py --config stress --alpha 0.0625 --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
$CMD1 > gpurun_out/stress_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_ns_gemm_tc_pair|k_splitk_reduce|k_gather_rows|k_scatter_cols_t|k_momentum_score|k_topk|k_col_scores" -s 20 -c 12 -o gpurun_out/stress_full $CMD1 > gpurun_out/stress_ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/stress_ncu_full.log
