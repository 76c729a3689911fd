#!/bin/bash
# Launch-option sweep (green_sms x lane_tiers) per workload; one summary line per run.
# usage: sweep_green.sh "<workload>:<greens>:<tiers>" ...   e.g. "big-newstest-8192w:0 24:20 30"
out=gpurun_out/sweep_green.txt; : > $out
for spec in "$@"; do
  IFS=: read w greens tiers <<< "$spec"
  for g in $greens; do for t in $tiers; do
    python bench.py --workload $w --green-sms $g --lane-tiers $t --steps 3 --no-cpu-baseline --no-roofline > gpurun_out/sw.log 2>&1
    python -c "import json;l=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]);print('$w', 'green', $g, 'tiers', $t, round(l['value']), round(l['ms_per_step'],2))" >> $out 2>&1 || tail -2 gpurun_out/sw.log >> $out
  done; done
done
cat $out
