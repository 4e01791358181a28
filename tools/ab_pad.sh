# A/B of the padded slab-major copies (FJ_ROWS_PAD_A / FJ_ROWS_PAD_B, rows.cuh), run under gpurun:
# product / loop time per variant (twice, interleaved), then the rows parity tests on each variant.
mkdir -p gpurun_out
bash tools/ab_rows.sh "c3 3" > gpurun_out/ab_rows_pad.log 2>&1
for L in paper_2101_08143_b200/variants/*.so; do
  echo "== $L" >> gpurun_out/ab_rows_pad_tests.log
  FJ_LIBRARY=$PWD/$L python -m pytest tests/test_gpu_rows.py -x -q 2>&1 | tail -3 >> gpurun_out/ab_rows_pad_tests.log
done
cat gpurun_out/ab_rows_pad.log; cat gpurun_out/ab_rows_pad_tests.log
