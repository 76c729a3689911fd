#!/bin/bash
mkdir -p gpurun_out/r2o
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -m gpu -k "attention or teacher_forced or self or big or config0 or long" > gpurun_out/r2o/tests.log 2>&1
for i in 1 2; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2o/bench_big_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self 1 > gpurun_out/r2o/bench_big_self1_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self 2 > gpurun_out/r2o/bench_big_self2_$i.json 2>/dev/null
done
for w in base-newstest-8192w; do for s in 0 1 2; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --attn-tma-self $s > gpurun_out/r2o/bench_${w}_self$s.json 2>/dev/null
done; done
for w in small-aan-newstest-8192w base-aan-newstest-8192w tiny192-aan-newstest-8192w; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2o/bench_$w.json 2>/dev/null
  MNMT_ATTN_TMA=0 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2o/bench_${w}_generic.json 2>/dev/null
done
python scripts/row_micro.py src > gpurun_out/r2o/attn_tma_box8.txt 2>&1
