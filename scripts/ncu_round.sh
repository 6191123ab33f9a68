#!/bin/bash
# ncu evidence for one snapshot (outputs in gpurun_out/): the launch list of the
# bench command, K7 DRAM traffic per launch, and --set full captures of the
# tensor-core K7 (level 7 -> 6) and K6 (level 8) at cfg4.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1; echo "ncu launches rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_upward -c 7 --csv --log-file gpurun_out/traffic_$TAG.csv python scripts/prof_run.py cfg4 > gpurun_out/ncu_traffic_$TAG.log 2>&1; echo "ncu traffic rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_upward_tc --launch-skip 3 -c 1 -f -o gpurun_out/tc_$TAG python scripts/prof_run.py cfg4 > gpurun_out/ncu_tc_$TAG.log 2>&1; echo "ncu tc rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_cousin_ws --launch-skip 2 -c 1 -f -o gpurun_out/cou_$TAG python scripts/prof_run.py cfg4 > gpurun_out/ncu_cou_$TAG.log 2>&1; echo "ncu cou rc=$?"
