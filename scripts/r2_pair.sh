#!/bin/bash
# CTA-pair persistent GEMM: parity, micro (encoder / output shapes), job A/B
mkdir -p gpurun_out/pair
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pair/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "pair" > gpurun_out/pair/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/pair/tests.log
timeout 600 python scripts/pair_micro.py > gpurun_out/pair/micro.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/pair/$n.json 2>/dev/null; }
run big_def
MNMT_PERS2=1 run big_p2
run baseaan_def --workload base-aan-newstest-8192w
MNMT_PERS2=1 run baseaan_p2 --workload base-aan-newstest-8192w
run small_def --workload small-aan-newstest-8192w
MNMT_PERS2=1 run small_p2 --workload small-aan-newstest-8192w
MNMT_PERS2=1 run big_p2_b
run big_def_b
