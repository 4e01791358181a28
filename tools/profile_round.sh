#!/bin/bash
# Profiling artefacts for profiles/ (run under gpurun on ONE GPU).
#  1. the bench command, plain (must exit 0 before ncu runs it)
#  2. ncu launch list (gpu__time_duration per launch) of the same command
#  3. ncu --set full of the dominant kernel (the PCG product of the bench workload), one launch,
#     recorded into profiles/ncu_traffic.json under (config, k, order, source hash)
# Usage: bash tools/profile_round.sh <config> <k> <tag> <kernel regex> [order]
set -u
CFG=${1:-c3}
K=${2:-3}
TAG=${3:-r02}
KREGEX=${4:-ApplyOpV}
ORDER=${5:-natural}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cuda-graph --spmv-reps 3 --vertex-order $ORDER --no-extras"
mkdir -p gpurun_out
$CMD > gpurun_out/prof_bench_plain_$CFG.json 2> gpurun_out/prof_bench_plain_$CFG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$CFG.csv $CMD \
    > gpurun_out/ncu_launch_$CFG.log 2>&1
echo "launch list rc=$?" >> gpurun_out/ncu_launch_$CFG.log
PCMD="python tools/spmv_variants.py --config $CFG --k $K --reps 3 --order $ORDER"
$PCMD > gpurun_out/prof_spmv_plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$KREGEX -s 1 -c 1 \
    -o gpurun_out/full_${TAG}_${CFG}_k$K $PCMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_$CFG.log
