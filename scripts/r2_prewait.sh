#!/bin/bash
mkdir -p gpurun_out/prewait
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/prewait/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/prewait/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/prewait/gpu_tests.log
timeout 300 python scripts/attn_f32_micro.py > gpurun_out/prewait/attn_micro.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/prewait/$n.json 2>/dev/null; }
for i in a b; do
run big_$i
run small_$i --workload small-aan-newstest-8192w
run baseaan_$i --workload base-aan-newstest-8192w
run base_$i --workload base-newstest-8192w
done
PRESET=big T=64 BS=1,16,64,256 timeout 900 python scripts/step_latency.py sab=64 smallm=0 attn_tma_self=2 > gpurun_out/prewait/step_big.txt 2>&1
