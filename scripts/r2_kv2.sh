#!/bin/bash
mkdir -p gpurun_out/kv2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/kv2/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > gpurun_out/kv2/tests.log 2>&1
echo "rc=$?" >> gpurun_out/kv2/tests.log
timeout 900 python -m pytest tests/test_gpu_model.py -q -x -k "self_attention_tma or big_student" >> gpurun_out/kv2/tests.log 2>&1
echo "model rc=$?" >> gpurun_out/kv2/tests.log
for v in 0 1; do MNMT_ATTN_KV2=$v timeout 300 python scripts/attn_f32_micro.py > gpurun_out/kv2/micro_kv2_$v.txt 2>&1; done
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/kv2/$n.json 2>/dev/null; }
MNMT_ATTN_KV2=0 run big_0
run big_1
MNMT_ATTN_KV2=0 run base_0 --workload base-newstest-8192w
run base_1 --workload base-newstest-8192w
MNMT_ATTN_KV2=0 run small_0 --workload small-aan-newstest-8192w
run small_1 --workload small-aan-newstest-8192w
MNMT_ATTN_KV2=0 run big_0b
run big_1b
