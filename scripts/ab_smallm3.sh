#!/bin/bash
# small-M path after the one-wave grid cap: row bound / K bound per workload.
set -u
run() { python bench.py --no-cpu-baseline --no-roofline --steps 5 "$@" | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=j['config']; print(c['workload'], 'smallm', c['smallm'], 'kmax', c['smallm_kmax'], round(j['value']), 'words/s', round(j['ms_per_step'],2), 'ms')"; }
for r in 1 2; do
  run --smallm 0; run --smallm 32 --smallm-kmax 512; run --smallm 32 --smallm-kmax 2048
  run --workload base-newstest-8192w --smallm 0; run --workload base-newstest-8192w --smallm 32
  run --workload base-aan-newstest-8192w --smallm 0; run --workload base-aan-newstest-8192w --smallm 32 --smallm-kmax 2048
done
