#!/bin/bash
mkdir -p gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3; do for v in 0 1; do
  MNMT_SPLITK=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2i/bench_splitk${v}_$i.json 2>/dev/null
done; done
PRESET=big GREEN=0 TIERS=25 python scripts/tier_probe.py > gpurun_out/r2i/tier_probe_big.txt 2>&1
SMALLM=1 python scripts/gemm_micro.py 1024 4096 > gpurun_out/r2i/gemm_big_smallm.txt 2>&1
for g in 0 24 40; do for t in 25 35; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --green-sms $g --lane-tiers $t > gpurun_out/r2i/bench_g${g}_t${t}.json 2>/dev/null
done; done
