# quantities pass / ttq: rows operator kernel (default) vs the merge-path engine (FJ_ROWS=0)
for cfg in "c3 3 natural" "c2 1 natural" "c3 1 natural" "c5 1 degree"; do
  set -- $cfg
  for m in -1 0; do
    FJ_ROWS=$m python tools/spmv_variants.py --config $1 --k $2 --reps 5 --order $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 k=$2 $3 FJ_ROWS=$m', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), 'quant_ms', round(d['quant_ms'],3), d['iters'], d['rel_res'], d['D0'])"
  done
done
