#!/bin/bash
mkdir -p gpurun_out/r2v
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PRESET=big LMAX=45 OPTS="lanes=2,lane_tiers=25,pers_reserve=16,smallm=0" timeout 1200 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v/launches_bulk.csv python scripts/job_once.py > gpurun_out/r2v/job_bulk.log 2>&1
python scripts/launch_summary.py gpurun_out/r2v/launches_bulk.csv > gpurun_out/r2v/launches_bulk_summary.txt
PRESET=big LMIN=46 OPTS="lanes=1,lane_tiers=0,pers_reserve=0,smallm=0" timeout 1200 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v/launches_crit.csv python scripts/job_once.py > gpurun_out/r2v/job_crit.log 2>&1
python scripts/launch_summary.py gpurun_out/r2v/launches_crit.csv > gpurun_out/r2v/launches_crit_summary.txt
for t in 15 25 35; do for g in 0 32; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --lane-tiers $t --green-sms $g > gpurun_out/r2v/bench_t${t}_g$g.json 2>/dev/null
done; done
for l in 2 4; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --lanes $l > gpurun_out/r2v/bench_lanes$l.json 2>/dev/null; done
