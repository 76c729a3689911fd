#!/bin/bash
mkdir -p gpurun_out/bigbox
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bigbox/build.log 2>&1
MNMT_BIGBOX=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/bigbox/tests.log 2>&1
echo "rc=$?" >> gpurun_out/bigbox/tests.log
for v in 0 1; do MNMT_BIGBOX=$v timeout 600 python scripts/gemm_micro.py 1024 4096 > gpurun_out/bigbox/micro_big_$v.txt 2>&1; done
for v in 0 1; do MNMT_BIGBOX=$v timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/bigbox/micro_small_$v.txt 2>&1; done
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/bigbox/$n.json 2>/dev/null; }
MNMT_BIGBOX=0 run big_0
MNMT_BIGBOX=1 run big_1
MNMT_BIGBOX=0 run small_0 --workload small-aan-newstest-8192w
MNMT_BIGBOX=1 run small_1 --workload small-aan-newstest-8192w
MNMT_BIGBOX=0 run baseaan_0 --workload base-aan-newstest-8192w
MNMT_BIGBOX=1 run baseaan_1 --workload base-aan-newstest-8192w
MNMT_BIGBOX=1 run big_1b
MNMT_BIGBOX=0 run big_0b
