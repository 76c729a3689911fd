#!/bin/bash
mkdir -p gpurun_out/r2q
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -m gpu -k "attention or teacher_forced or self or big or long" > gpurun_out/r2q/tests.log 2>&1
python scripts/row_micro.py src > gpurun_out/r2q/attn_tma_q.txt 2>&1
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2q/bench_big_$i.json 2>/dev/null
done
for w in small-aan-newstest-8192w base-aan-newstest-8192w base-newstest-8192w; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2q/bench_$w.json 2>/dev/null
done
