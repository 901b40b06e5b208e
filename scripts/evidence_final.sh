#!/bin/bash
# GPU suite + smoke + the round-end evidence, with the ncu reports summarised on the box and
# the raw .ncu-rep files removed (gpurun merges at most 64 MiB of gpurun_out/ back).
cd "$(dirname "$0")/.."
bash scripts/gpu_round.sh
NO_BENCH=1 bash scripts/evidence.sh
python scripts/summarize_ncu.py launches gpurun_out/launches.csv > gpurun_out/sum_launches.md 2> gpurun_out/sum_launches.err
python scripts/summarize_ncu.py full gpurun_out/prof.ncu-rep > gpurun_out/sum_full.md 2> gpurun_out/sum_full.err
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out > gpurun_out/du.txt
