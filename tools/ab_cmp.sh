#!/bin/bash
# A/B timing of two libfj.so builds (run under gpurun): solve loop, product and quantities-pass
# times per config, alternating builds twice.  A = $1 (default the committed-HEAD copy built into
# variants/libfj_head.so), B = the in-tree build.  Usage: bash tools/ab_cmp.sh [A.so] ["c3 3" "c4 64" ...]
A=${1:-paper_2101_08143_b200/variants/libfj_head.so}
shift || true
CFGS=("$@"); [ ${#CFGS[@]} -eq 0 ] && CFGS=("c3 3" "c4 64")
for i in 1 2; do
 for L in "$A" paper_2101_08143_b200/libfj.so; do
  for c in "${CFGS[@]}"; do set -- $c
   FJ_LIBRARY=$L python tools/spmv_variants.py --config $1 --k $2 --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L'[-24:], '$1', 'spmv', round(d['spmv_ms'],4), 'quant', round(d['quant_ms'],3), 'ttq', round(d['ms'],3), 'loop', round(d['loop_ms'],3), d['iters'], d['rel_res'])"
  done
 done
done
