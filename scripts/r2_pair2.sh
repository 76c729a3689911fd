#!/bin/bash
mkdir -p gpurun_out/pair2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pair2/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pair2/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/pair2/tests.log
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/pair2/$n.json 2>/dev/null; }
run big_rule
MNMT_PERS2=0 run big_off
run baseaan_rule --workload base-aan-newstest-8192w
MNMT_PERS2=0 run baseaan_off --workload base-aan-newstest-8192w
run small_rule --workload small-aan-newstest-8192w
MNMT_PERS2=0 run small_off --workload small-aan-newstest-8192w
run big_rule_b
MNMT_PERS2=0 run big_off_b
