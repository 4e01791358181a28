#!/bin/bash
# One gpurun call: GPU suite, default bench line, ncu launch list of the bench command, ncu --set full
# of ONE product (all its launches) with its DRAM traffic recorded under the build's source hash.
# Usage: bash tools/round_evidence.sh <tag> [kernel regex] [launches per product]
TAG=${1:-r02}
KREGEX=${2:-"k_rows<"}
NL=${3:-2}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --config c3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cuda-graph --spmv-reps 3 --no-extras"
$CMD > gpurun_out/prof_plain_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c3.csv $CMD \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?" >> gpurun_out/ncu_launch_$TAG.log
PCMD="python tools/spmv_variants.py --config c3 --k 3 --reps 3"
FJV_NO_GRAPH=1 $PCMD > gpurun_out/prof_spmv_plain_$TAG.log 2>&1 && \
FJV_NO_GRAPH=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$KREGEX \
    -s $NL -c $NL -o gpurun_out/full_${TAG}_c3_k3 $PCMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_$TAG.log
