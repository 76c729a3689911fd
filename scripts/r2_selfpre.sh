#!/bin/bash
mkdir -p gpurun_out/selfpre
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/selfpre/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/selfpre/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/selfpre/gpu_tests.log
for v in 0 1; do MNMT_ATTN_SELF_PRE=$v PRESET=big T=64 BS=1,16,64,256 timeout 900 python scripts/step_latency.py sab=64 smallm=0 attn_tma_self=2 > gpurun_out/selfpre/step_big_$v.txt 2>&1; done
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/selfpre/$n.json 2>/dev/null; }
for i in a b; do
MNMT_ATTN_SELF_PRE=0 run big_0$i
run big_1$i
MNMT_ATTN_SELF_PRE=0 run base_0$i --workload base-newstest-8192w
run base_1$i --workload base-newstest-8192w
done
