#!/bin/bash
mkdir -p gpurun_out/r2u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -m gpu -k "attention or teacher_forced or self or big or long" > gpurun_out/r2u/tests.log 2>&1
for i in 1 2; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2u/bench_big_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self 1 > gpurun_out/r2u/bench_big_self1_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self 2 > gpurun_out/r2u/bench_big_self2_$i.json 2>/dev/null
done
for s in 0 1 2; do
  python bench.py --workload base-newstest-8192w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self $s > gpurun_out/r2u/bench_base_self$s.json 2>/dev/null
done
PRESET=big GREEN=0 TIERS=25 python scripts/tier_probe.py > gpurun_out/r2u/tier_probe_big.txt 2>&1
