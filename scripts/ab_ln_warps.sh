#!/bin/bash
# A/B: rows (warps) per CTA of the LayerNorm kernel (env MNMT_LN_WARPS), headline bench, twice each
for rep in 1 2; do for w in 4 1 2; do
  MNMT_LN_WARPS=$w python bench.py --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/ab.log 2>&1
  python -c "import json;l=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('ln_warps $w', round(l['value']), round(l['ms_per_step'],2))"
done; done
for w in 4 1; do
  MNMT_LN_WARPS=$w BS=8,64,256 python scripts/step_latency.py 2>&1 | sed "s/^/ln_warps=$w /"
done
