set -u
mkdir -p gpurun_out
bash tools/profile_round.sh c2 1 r02 "ApplyOp<" natural
PCMD="python tools/spmv_variants.py --config c5 --k 1 --reps 3 --order degree"
$PCMD > gpurun_out/prof_spmv_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ApplyOp<" -s 1 -c 1 \
    -o gpurun_out/full_r02_c5_k1 $PCMD > gpurun_out/ncu_full_c5.log 2>&1
echo "full c5 rc=$?" >> gpurun_out/ncu_full_c5.log
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:QuantOp<" -s 0 -c 1 \
    -o gpurun_out/full_r02_c5_quant $PCMD > gpurun_out/ncu_full_c5q.log 2>&1
echo "full c5 quant rc=$?" >> gpurun_out/ncu_full_c5q.log
