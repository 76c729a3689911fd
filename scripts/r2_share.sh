#!/bin/bash
mkdir -p gpurun_out/r2t
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MNMT_ATTN_SHARE=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -m gpu -k "attention or teacher_forced or big" > gpurun_out/r2t/tests_share.log 2>&1
MNMT_ATTN_SHARE=1 python scripts/row_micro.py src > gpurun_out/r2t/attn_share.txt 2>&1
python scripts/row_micro.py src > gpurun_out/r2t/attn_sep.txt 2>&1
for i in 1 2; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2t/bench_big_sep_$i.json 2>/dev/null
  MNMT_ATTN_SHARE=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2t/bench_big_share_$i.json 2>/dev/null
done
for w in small-aan-newstest-8192w base-aan-newstest-8192w; do
  MNMT_ATTN_SHARE=1 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2t/bench_${w}_share.json 2>/dev/null
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2t/bench_${w}_sep.json 2>/dev/null
done
