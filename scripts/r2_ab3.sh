#!/bin/bash
mkdir -p gpurun_out/r2m
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local tag=$1; shift; env "$@" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2m/bench_$tag.json 2>/dev/null; }
for i in 1 2; do
  run srcsplit_$i MNMT_ATTN_TMA_SELF=0 MNMT_ENC_R64=0
  run selfsplit_$i MNMT_ATTN_TMA_SELF=1 MNMT_ENC_R64=0
  run selfsplit_enc_$i MNMT_ATTN_TMA_SELF=1
done
for w in base-newstest-8192w base-aan-newstest-8192w small-aan-newstest-8192w tiny192-aan-newstest-8192w; do
  for v in "MNMT_ATTN_TMA=0 MNMT_ENC_R64=0" "MNMT_ATTN_TMA_SELF=1 MNMT_ENC_R64=0" "MNMT_ATTN_TMA_SELF=0 MNMT_ENC_R64=0"; do
    tag=$(echo $v | tr ' =' '__')
    env $v python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2m/bench_${w}_$tag.json 2>/dev/null
  done
done
