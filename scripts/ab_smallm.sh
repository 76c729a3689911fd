#!/bin/bash
# A/B of the small-M GEMM path (IDP4A at <= "smallm" live rows) against tcgen05 everywhere:
# per-step latency at 1-32 rows, then the configs[1] job (and base-AAN, big) per row bound.
set -u
for b in 0 32; do
  echo "smallm=$b"; BS=1,8,16,32 python scripts/step_latency.py smallm=$b
done
for wl in "" "--workload base-aan-newstest-8192w" "--workload big-newstest-8192w"; do
  for b in 0 8 16 32 0 8 16; do
    MNMT_SMALLM=$b python bench.py --no-cpu-baseline --no-roofline $wl | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('smallm', $b, j['config']['workload'], round(j['value']), 'words/s', round(j['ms_per_step'],2), 'ms')"
  done
done
