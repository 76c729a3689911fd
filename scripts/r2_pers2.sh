#!/bin/bash
mkdir -p gpurun_out/pers2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pers2/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pers2/tests.log 2>&1
echo "rc=$?" >> gpurun_out/pers2/tests.log
timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/pers2/micro_small.txt 2>&1
MNMT_BN32=0 timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/pers2/micro_small_nobn32.txt 2>&1
MNMT_BN32=0 timeout 600 python scripts/gemm_micro.py 512 2048 > gpurun_out/pers2/micro_base_nobn32.txt 2>&1
timeout 600 python scripts/gemm_micro.py 512 2048 > gpurun_out/pers2/micro_base.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/pers2/$n.json 2>/dev/null; }
run big
MNMT_GEMM_PERSISTENT=0 run big_old
run small --workload small-aan-newstest-8192w
MNMT_BN32=0 run small_nobn32 --workload small-aan-newstest-8192w
run baseaan --workload base-aan-newstest-8192w
MNMT_BN32=0 run baseaan_nobn32 --workload base-aan-newstest-8192w
run base --workload base-newstest-8192w
run tiny --workload tiny192-aan-newstest-8192w
run big_b
