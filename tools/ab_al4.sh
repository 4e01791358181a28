# A/B of the aligned-group index loads (FJ_ROWS_AL4, rows.cuh), run under gpurun: C3 k = 3 (slab-B
# pass), C2 / C5 k = 1 (one-pass kernel), then the rows parity tests on the variant.
mkdir -p gpurun_out
bash tools/ab_rows.sh "c3 3" > gpurun_out/ab_rows_al4.log 2>&1
for cfg in "c2 natural" "c5 degree" "c3 natural"; do
  set -- $cfg
  for L in paper_2101_08143_b200/libfj.so paper_2101_08143_b200/variants/*.so; do
    FJ_LIBRARY=$L python tools/spmv_variants.py --config $1 --k 1 --reps 5 --order $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 k=1 $(basename $L)', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), d['iters'], d['rel_res'])" >> gpurun_out/ab_rows_al4.log
  done
done
for L in paper_2101_08143_b200/variants/*.so; do
  echo "== $L" >> gpurun_out/ab_rows_al4.log
  FJ_LIBRARY=$PWD/$L python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3 >> gpurun_out/ab_rows_al4.log
done
cat gpurun_out/ab_rows_al4.log
