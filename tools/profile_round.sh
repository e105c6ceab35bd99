#!/bin/bash
# Round profiling: plain bench line, ncu launch list of one c5 step, full ncu
# captures of the top kernels.  Run under gpurun; outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1200 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log
python tools/profile_step.py c5 > gpurun_out/plain_c5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
      python tools/profile_step.py c5 > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_pmc|k_brick_posterior" -c 2 \
    -o gpurun_out/prof_c5_leaf python tools/profile_step.py c5 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_marginals" --launch-skip 8 -c 1 \
    -o gpurun_out/prof_c5_marg python tools/profile_step.py c5 > gpurun_out/ncu_marg.log 2>&1; echo "ncu marg rc=$?"
