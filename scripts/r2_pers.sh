#!/bin/bash
mkdir -p gpurun_out/pers
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pers/build.log 2>&1
MNMT_GEMM_PERSISTENT=1 timeout 600 python scripts/gemm_micro.py 1024 4096 > gpurun_out/pers/micro_big_p1.txt 2>&1
MNMT_GEMM_PERSISTENT=1 timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/pers/micro_small_p1.txt 2>&1
timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/pers/micro_small_p0.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/pers/$n.json 2>/dev/null; }
run big_def
MNMT_GEMM_PERSISTENT=1 run big_p1
run small_def --workload small-aan-newstest-8192w
MNMT_GEMM_PERSISTENT=1 run small_p1 --workload small-aan-newstest-8192w
run baseaan_def --workload base-aan-newstest-8192w
MNMT_GEMM_PERSISTENT=1 run baseaan_p1 --workload base-aan-newstest-8192w
MNMT_GEMM_PERSISTENT=1 run big_p1_b
run big_def_b
