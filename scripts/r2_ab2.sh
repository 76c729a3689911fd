#!/bin/bash
mkdir -p gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local tag=$1; shift; env "$@" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2l/bench_$tag.json 2>/dev/null; }
for i in 1 2; do
  run old_$i MNMT_ATTN_TMA=0 MNMT_ENC_R64=0
  run src_$i MNMT_ATTN_TMA_SELF=0 MNMT_ATTN_TMA_SPLIT=0 MNMT_ENC_R64=0
  run srcsplit_$i MNMT_ATTN_TMA_SELF=0 MNMT_ENC_R64=0
  run srcself_$i MNMT_ATTN_TMA_SPLIT=0 MNMT_ENC_R64=0
  run all_$i MNMT_ENC_R64=0
  run src_enc_$i MNMT_ATTN_TMA_SELF=0 MNMT_ATTN_TMA_SPLIT=0
done
for v in "MNMT_ATTN_TMA=0 MNMT_ENC_R64=0" "MNMT_ATTN_TMA_SELF=0 MNMT_ATTN_TMA_SPLIT=0 MNMT_ENC_R64=0" "MNMT_ENC_R64=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v PRESET=big GREEN=0 TIERS=25 python scripts/tier_probe.py > gpurun_out/r2l/tier_$tag.txt 2>&1
done
MNMT_SPLITK=0 timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "gemm or attention or gather" -p no:cacheprovider > gpurun_out/r2l/synccheck.kernels.log 2>&1
echo "rc=$?" >> gpurun_out/r2l/synccheck.kernels.log
