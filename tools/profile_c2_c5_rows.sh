# ncu --set full of ONE k = 1 product on the lean row kernels (k_rows_chunks + k_rows<PASS 2>) for C2
# (natural order) and C5 (degree order), and of the C5 fused quantities pass (k_op_chunks +
# k_op_rows<QuantOp>), run under gpurun; host-driven loop (ncu cannot see conditional graph bodies).
set -u
mkdir -p gpurun_out
export FJV_NO_GRAPH=1
for co in "c2 natural" "c5 degree"; do
  set -- $co
  PCMD="python tools/spmv_variants.py --config $1 --k 1 --reps 3 --order $2"
  $PCMD > gpurun_out/prof_rows_plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_rows(<|_chunks)" -s 2 -c 2 \
      -o gpurun_out/full_rows_$1_k1 $PCMD > gpurun_out/ncu_full_rows_$1.log 2>&1
  echo "full $1 rc=$?" >> gpurun_out/ncu_full_rows_$1.log
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:QuantOp" -s 0 -c 2 \
    -o gpurun_out/full_rows_c5_quant $PCMD > gpurun_out/ncu_full_rows_c5q.log 2>&1
echo "full c5 quant rc=$?" >> gpurun_out/ncu_full_rows_c5q.log
tail -2 gpurun_out/ncu_full_rows_*.log gpurun_out/prof_rows_plain_*.log
