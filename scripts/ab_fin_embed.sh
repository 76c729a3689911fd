#!/bin/bash
# A/B of the fin_embed option (next step's embedding inside k_finish): per-step latency at
# several row counts, then the configs[1] job with the option off / at 128 / 512 rows.
set -u
mkdir -p gpurun_out
for fe in 0 128 1048576; do
  echo "fin_embed=$fe"; BS=8,128,512,2048 python scripts/step_latency.py fin_embed=$fe
done
for fe in 0 128 512 0 128; do
  python bench.py --no-cpu-baseline --no-roofline --fin-embed $fe | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fin_embed', $fe, round(j['value']), 'words/s', round(j['ms_per_step'],2), 'ms', 'launches', j['gpu_launches'])"
done
