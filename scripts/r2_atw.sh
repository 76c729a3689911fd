#!/bin/bash
mkdir -p gpurun_out/atw
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/atw/build.log 2>&1
for w in 2 8; do MNMT_AT_WARPS=$w timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "src_attention" >> gpurun_out/atw/tests.log 2>&1; echo "w$w rc=$?" >> gpurun_out/atw/tests.log; done
for w in 2 4 8; do MNMT_AT_WARPS=$w timeout 300 python scripts/attn_f32_micro.py > gpurun_out/atw/micro_w$w.txt 2>&1; done
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/atw/$n.json 2>/dev/null; }
run big_w4
MNMT_AT_WARPS=8 run big_w8
MNMT_AT_WARPS=2 run big_w2
run base_w4 --workload base-newstest-8192w
MNMT_AT_WARPS=8 run base_w8 --workload base-newstest-8192w
run small_w4 --workload small-aan-newstest-8192w
MNMT_AT_WARPS=8 run small_w8 --workload small-aan-newstest-8192w
MNMT_AT_WARPS=8 run big_w8_b
run big_w4_b
