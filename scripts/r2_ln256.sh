#!/bin/bash
mkdir -p gpurun_out/ln256
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ln256/build.log 2>&1
MNMT_LN_SPLIT256=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" > gpurun_out/ln256/tests.log 2>&1
echo "rc=$?" >> gpurun_out/ln256/tests.log
for v in 0 1; do
  MNMT_LN_SPLIT256=$v PRESET=small-aan T=48 BS=1,64,632 timeout 900 python scripts/step_latency.py smallm=32 smallm_kmax=2048 attn_tma_self=2 > gpurun_out/ln256/step_s$v.txt 2>&1
done
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/ln256/$n.json 2>/dev/null; }
run small_s0 --workload small-aan-newstest-8192w
MNMT_LN_SPLIT256=1 run small_s1 --workload small-aan-newstest-8192w
run small_s0_b --workload small-aan-newstest-8192w
MNMT_LN_SPLIT256=1 run small_s1_b --workload small-aan-newstest-8192w
