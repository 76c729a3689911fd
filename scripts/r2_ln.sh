#!/bin/bash
# LN one-float4-per-thread A/B (step latency + job), GEMM chain timeline, lanes / tiers sweep
mkdir -p gpurun_out/ln2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ln2/build.log 2>&1
MNMT_LN_NV1=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" > gpurun_out/ln2/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ln2/tests.log
for v in 0 1; do
  MNMT_LN_NV1=$v PRESET=big T=48 BS=1,64,632 timeout 900 python scripts/step_latency.py sab=64 smallm=0 attn_tma_self=2 > gpurun_out/ln2/step_nv$v.txt 2>&1
done
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/ln2/$n.json 2>/dev/null; }
run big_nv0
MNMT_LN_NV1=1 run big_nv1
MNMT_LN_NV1=1 run baseaan_nv1 --workload base-aan-newstest-8192w
run baseaan_nv0 --workload base-aan-newstest-8192w
run big_t10 --lane-tiers 10
run big_t20 --lane-tiers 20
run big_l3t15 --lanes 3 --lane-tiers 15
run big_l3t30 --lanes 3 --lane-tiers 30
run big_sab128 --sab 128
MNMT_LN_NV1=1 run big_nv1_b
run big_nv0_b
SHAPES="8x1024x1024,64x1024x1024,630x1024x1024,8x1024x4096,8x4096x1024" timeout 600 python scripts/gemm_chain.py > gpurun_out/ln2/gemm_chain.txt 2>&1
# fp32 attention measurement variant (MNMT_ATTN_F32=1; departs from R20, timing only)
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "src_attention_tma" >> gpurun_out/ln2/tests.log 2>&1
echo "attn tests rc=$?" >> gpurun_out/ln2/tests.log
KERNEL=attn D=1024 H=16 M=630 S=21 timeout 300 python scripts/attn_f32_micro.py > gpurun_out/ln2/attn_f64.txt 2>&1
MNMT_ATTN_F32=1 KERNEL=attn timeout 300 python scripts/attn_f32_micro.py > gpurun_out/ln2/attn_f32.txt 2>&1
MNMT_ATTN_F32=1 run big_attnf32
