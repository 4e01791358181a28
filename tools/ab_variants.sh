#!/bin/bash
# A/B of libfj.so tuning variants (run under gpurun): PCG product / loop time per variant, twice.
# Usage: bash tools/ab_variants.sh "<config> <k>" [variant.so ...]   (default variants: variants/*.so)
CFG=${1:-"c3 3"}; shift || true
VS=("$@"); [ ${#VS[@]} -eq 0 ] && VS=(paper_2101_08143_b200/libfj.so paper_2101_08143_b200/variants/*.so)
set -- $CFG
for i in 1 2; do
  for L in "${VS[@]}"; do
    FJ_LIBRARY=$L python tools/spmv_variants.py --config $1 --k $2 --reps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', 'spmv', round(d['spmv_ms'],4), 'loop', round(d['loop_ms'],3), 'ttq', round(d['ms'],3), d['iters'], d['rel_res'])"
  done
done
