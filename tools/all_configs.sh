#!/bin/bash
# Bench line of every configuration (run under gpurun): gpurun_out/${TAG}_bench_<cfg>.json
TAG=${1:-r2}
mkdir -p gpurun_out
for w in c1 c2 c3 c4 p1; do
  python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
python bench.py --workload c3 --dense exact > gpurun_out/${TAG}_bench_c3_dense.json 2> gpurun_out/${TAG}_bench_c3_dense.err
python bench.py --workload c4 --separate-iso --no-cpu-baseline > gpurun_out/${TAG}_bench_c4_separate.json 2> gpurun_out/${TAG}_bench_c4_separate.err
python bench.py --workload x1024 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_x1024.json 2> gpurun_out/${TAG}_bench_x1024.err
python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG}_reference_c5.json 2> gpurun_out/${TAG}_reference_c5.err
