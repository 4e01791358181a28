#!/bin/bash
# Profiling artefacts for profiles/ (run under gpurun on ONE GPU).
#  1. the bench command, plain (must exit 0 before ncu runs it)
#  2. ncu launch list (gpu__time_duration per launch) of the same command
#  3. ncu --set full of the dominant kernel (the (I+L)p warp-engine SpMV), one launch
set -u
CFG=${1:-c3}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cuda-graph --spmv-reps 3"
mkdir -p gpurun_out
$CMD > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD \
    > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/ncu_launch.log
python tools/prof_spmv.py --config $CFG --reps 3 > gpurun_out/prof_spmv_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'warp_kernel<0, fj::ApplyOp' -s 3 -c 1 \
    -o gpurun_out/spmv_full_$CFG python tools/prof_spmv.py --config $CFG --reps 3 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
