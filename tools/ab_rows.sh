# A/B of the rows-product tuning variants (run under gpurun): product / loop time per variant, twice
CFG=${1:-"c3 3"}; set -- $CFG
for i in 1 2; do
  for L in paper_2101_08143_b200/libfj.so paper_2101_08143_b200/variants/*.so; do
    FJ_LIBRARY=$L python tools/spmv_variants.py --config $1 --k $2 --reps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), d['iters'], d['rel_res'])"
  done
done
