#!/bin/bash
# Round-2 first probe: launch lists of one big / base-aan job (ncu, serialised, shares only)
# plus the bench line of the big workload.
set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2/smoke.log 2>&1
python bench.py --workload big-newstest-8192w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_big.json 2> gpurun_out/r2/bench_big.err
for P in big; do
  PRESET=$P OPTS="lanes=3,lane_tiers=25,pers_reserve=16,smallm=0" timeout 1200 ncu --nvtx --nvtx-include "job/" --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/r2/launches_$P.csv python scripts/job_once.py > gpurun_out/r2/job_$P.log 2>&1
  python scripts/launch_summary.py gpurun_out/r2/launches_$P.csv > gpurun_out/r2/launches_${P}_summary.txt
done
