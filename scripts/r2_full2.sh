#!/bin/bash
# Full check of the current build + the bulk tiers' launch list (big) + synccheck without -x.
mkdir -p gpurun_out/r2n
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2n/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2n/gpu_tests.log 2>&1
cp gpurun_out/parity/r2_parity.jsonl gpurun_out/r2n/ 2>/dev/null
python bench.py > gpurun_out/r2n/bench.json 2> gpurun_out/r2n/bench.err
PRESET=big LMAX=45 OPTS="lanes=2,lane_tiers=25,pers_reserve=16,smallm=0" timeout 1200 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n/launches_bulk.csv python scripts/job_once.py > gpurun_out/r2n/job_bulk.log 2>&1
python scripts/launch_summary.py gpurun_out/r2n/launches_bulk.csv > gpurun_out/r2n/launches_bulk_summary.txt
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -m gpu \
  -k "not test_gemm_split_k_acc_bitexact[257-1024-1024-64-8]" -p no:cacheprovider > gpurun_out/r2n/synccheck.kernels.log 2>&1
echo "rc=$?" >> gpurun_out/r2n/synccheck.kernels.log
