# A/B of the slab-major column copies (FJ_ROWS_SPLIT) on one box: product / loop /
# ttq per setting (C3 k = 3, C2 k = 3 forced to two slabs), alternating, three rounds; then bench.
for i in 1 2 3; do
  for s in 0 1; do
    FJ_ROWS_SPLIT=$s python tools/spmv_variants.py --config c3 --k 3 --reps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 k=3 FJ_ROWS_SPLIT=$s', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), d['iters'], d['rel_res'])"
  done
done
for s in 0 1 0 1; do
  FJ_ROWS_SPLIT=$s python bench.py --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench FJ_ROWS_SPLIT=$s', d['value'], d['unit'], 'ms_per_step', d['ms_per_step'], 'ttq', d.get('time_to_quantities_ms'), 'product', d['roofline']['launch_ms'])"
done
