#!/bin/bash
# finer encoder length buckets A/B; full GPU test suite on the new defaults
mkdir -p gpurun_out/fine
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fine/smoke.log 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/fine/$n.json 2>/dev/null; }
run big_fine
MNMT_ENC_FINE=0 run big_coarse
run base-aan_fine --workload base-aan-newstest-8192w
MNMT_ENC_FINE=0 run base-aan_coarse --workload base-aan-newstest-8192w
run small-aan_fine --workload small-aan-newstest-8192w
MNMT_ENC_FINE=0 run small-aan_coarse --workload small-aan-newstest-8192w
run big_fine_b
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/fine/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/fine/gpu_tests.log
