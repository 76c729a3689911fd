#!/bin/bash
# warp-uniform elect MMA issue: parity, micro, chain timeline, jobs
mkdir -p gpurun_out/elect
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/elect/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/elect/tests.log 2>&1
echo "rc=$?" >> gpurun_out/elect/tests.log
timeout 600 python scripts/gemm_micro.py 1024 4096 > gpurun_out/elect/micro_big.txt 2>&1
timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/elect/micro_small.txt 2>&1
ROWS=1,16,32,64 timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/elect/sab_micro_big.txt 2>&1
SHAPES="8x1024x1024,64x1024x1024,630x1024x1024,8x1024x4096,8x256x256" timeout 600 python scripts/gemm_chain.py > gpurun_out/elect/gemm_chain.txt 2>&1
timeout 600 python scripts/pair_micro.py > gpurun_out/elect/pair_micro.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/elect/$n.json 2>/dev/null; }
run big
run small --workload small-aan-newstest-8192w
run baseaan --workload base-aan-newstest-8192w
run base --workload base-newstest-8192w
run tiny --workload tiny192-aan-newstest-8192w
run big_b
