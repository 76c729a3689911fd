#!/bin/bash
mkdir -p gpurun_out/r2s
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_beam.py -x -q -m gpu > gpurun_out/r2s/tests.log 2>&1
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2s/bench_big_$i.json 2>/dev/null
done
for w in small-aan-newstest-8192w base-aan-newstest-8192w base-newstest-8192w tiny192-aan-newstest-8192w; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2s/bench_$w.json 2>/dev/null
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self 1 > gpurun_out/r2s/bench_big_self1.json 2>/dev/null
python bench.py --workload base-newstest-8192w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self 1 > gpurun_out/r2s/bench_base_self1.json 2>/dev/null
