# A/B of the k = 1 rows-product variants (run under gpurun): product / loop time per variant
for cfg in "c2 natural" "c3 natural" "c5 natural" "c5 degree"; do
  set -- $cfg
  for L in paper_2101_08143_b200/libfj.so paper_2101_08143_b200/variants/*.so; do
    for m in 1; do
      FJ_ROWS=$m FJ_LIBRARY=$L python tools/spmv_variants.py --config $1 --k 1 --reps 5 --order $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $(basename $L) FJ_ROWS=$m', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), d['iters'], d['rel_res'])"
    done
  done
  FJ_ROWS=0 python tools/spmv_variants.py --config $1 --k 1 --reps 5 --order $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 engine', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), d['iters'], d['rel_res'])"
done
