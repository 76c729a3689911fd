#!/bin/bash
# small-M path with its K bound (smallm_kmax 512): job A/B per workload, bound 0 vs 32.
set -u
for wl in small-aan-newstest-8192w base-aan-newstest-8192w base-newstest-8192w big-newstest-8192w tiny192-aan-newstest-8192w; do
  for b in 0 32 0 32; do
    MNMT_SMALLM=$b python bench.py --no-cpu-baseline --no-roofline --workload $wl --steps 5 | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('smallm', $b, j['config']['workload'], round(j['value']), 'words/s', round(j['ms_per_step'],2), 'ms')"
  done
done
