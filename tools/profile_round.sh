#!/bin/bash
# Round profiling (run under gpurun): plain bench line, ncu launch list of one c5
# step, full ncu captures of the top kernels.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
python tools/profile_step.py c5 > gpurun_out/plain_c5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
      python tools/profile_step.py c5 > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/pmc_variants.py one 4194304 > gpurun_out/plain_pmc.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_pmc" -c 1 \
      -o gpurun_out/prof_c5_pmc python tools/pmc_variants.py one 4194304 > gpurun_out/ncu_pmc.log 2>&1; echo "ncu pmc rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_brick" -c 1 \
    -o gpurun_out/prof_c5_brick python tools/profile_step.py c5 > gpurun_out/ncu_brick.log 2>&1; echo "ncu brick rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_marginals|k_bucket_factor" -c 2 \
    -o gpurun_out/prof_c5_fit python tools/profile_step.py c5 > gpurun_out/ncu_fit.log 2>&1; echo "ncu fit rc=$?"
