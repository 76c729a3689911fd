#!/bin/bash
# Round-end measurements on one B200: the headline bench line, every BASELINE config, the F1-F3
# lines, and an ncu launch list of one headline job.
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
for w in tiny192-aan-newstest-8192w base-aan-newstest-8192w base-newstest-8192w big-newstest-8192w; do
  python bench.py --workload $w --steps 5 >> gpurun_out/final/configs.jsonl 2>> gpurun_out/final/configs.err
done
python bench.py --shortlist --steps 5 > gpurun_out/final/shortlist.json 2>&1
python bench.py --kv-bf16 --steps 5 > gpurun_out/final/kvbf16.json 2>&1
python bench.py --beam 2 --steps 3 > gpurun_out/final/beam2.json 2>&1
ncu --nvtx --nvtx-include "job/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/final/job_launches.csv python scripts/job_once.py > gpurun_out/final/ncu_job.log 2>&1
python scripts/launch_summary.py gpurun_out/final/job_launches.csv > gpurun_out/final/job_launches_summary.txt 2>&1
tail -c 300 gpurun_out/final/bench.json; echo; wc -l gpurun_out/final/configs.jsonl; head -12 gpurun_out/final/job_launches_summary.txt
