#!/bin/bash
# bench.py flag sets, one summary line each:  sweep_opts.sh "<flags>" "<flags>" ...
out=gpurun_out/sweep_opts.txt; : > $out
for f in "$@"; do
  python bench.py $f --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/so.log 2>&1
  python -c "import json;l=json.loads(open('gpurun_out/so.log').read().strip().splitlines()[-1]);print('$f |', round(l['value']), round(l['ms_per_step'],2))" >> $out 2>&1 || tail -2 gpurun_out/so.log >> $out
done
cat $out
