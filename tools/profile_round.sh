#!/bin/bash
# Round profiling (run under gpurun): plain bench line, ncu launch list of the bench
# command, full ncu captures of the top kernels.  Outputs land in gpurun_out/ (scratch);
# summaries are copied to profiles/ by hand (tools/launch_summary.py, tools/ncu_summary.py).
#   bash tools/profile_round.sh [TAG]      (TAG defaults to r2)
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
# 1. the bench line (no profiler)
python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err; echo "bench rc=$?"
# 2. launch list of the same command (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c5.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
# 3. full captures of the dominant kernels (one launch each)
python tools/pmc_variants.py one 4194304 > gpurun_out/plain_pmc.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_pmc" -c 1 \
      -o gpurun_out/${TAG}_prof_c5_pmc python tools/pmc_variants.py one 4194304 > gpurun_out/ncu_pmc.log 2>&1
echo "ncu pmc rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_brick|k_chol8_rec" -c 2 \
    -o gpurun_out/${TAG}_prof_c5_brick python tools/profile_step.py c5 > gpurun_out/ncu_brick.log 2>&1
echo "ncu brick rc=$?"
