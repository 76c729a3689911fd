#!/bin/bash
mkdir -p gpurun_out/sync2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sync2/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/sync2/tests.log 2>&1
echo "rc=$?" >> gpurun_out/sync2/tests.log
ROWS=1,16,32,64 timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/sync2/sab_micro.txt 2>&1
ROWS=1,8,32 timeout 600 python scripts/sab_micro.py 256 2048 > gpurun_out/sync2/sab_micro_small.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/sync2/$n.json 2>/dev/null; }
run big
run small --workload small-aan-newstest-8192w
run baseaan --workload base-aan-newstest-8192w
run base --workload base-newstest-8192w
run tiny --workload tiny192-aan-newstest-8192w
MNMT_NPSYNC=0 run big_np0
run big_b
