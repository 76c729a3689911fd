#!/bin/bash
# Where the big job's critical tier spends its time: per-step latency vs rows, and the ncu launch
# list of the critical tier (sentences of 28..100 words) decoded alone.
mkdir -p gpurun_out/crit
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/crit/build.log 2>&1
PRESET=big T=64 BS=1,16,32,64,128,256,632 timeout 900 python scripts/step_latency.py sab=64 smallm=0 attn_tma_self=2 > gpurun_out/crit/step_latency_s64.txt 2>&1
PRESET=big T=64 BS=1,16,64,256 timeout 900 python scripts/step_latency.py smallm=32 smallm_kmax=1024 attn_tma_self=2 > gpurun_out/crit/step_latency_def.txt 2>&1
PRESET=big LMIN=28 OPTS="lanes=1,pers_reserve=0,smallm=0,sab=64,attn_tma_self=2" timeout 1200 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/crit/launches_crit.csv python scripts/job_once.py > gpurun_out/crit/job_crit.log 2>&1
python scripts/launch_summary.py gpurun_out/crit/launches_crit.csv > gpurun_out/crit/launches_crit_summary.txt
PRESET=big LMAX=27 OPTS="lanes=1,pers_reserve=0,smallm=0,sab=64,attn_tma_self=2" timeout 1200 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/crit/launches_bulk.csv python scripts/job_once.py > gpurun_out/crit/job_bulk.log 2>&1
python scripts/launch_summary.py gpurun_out/crit/launches_bulk.csv > gpurun_out/crit/launches_bulk_summary.txt
rm -f gpurun_out/crit/launches_*.csv
