#!/bin/bash
mkdir -p gpurun_out/r2j
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/r2j/kernels.log 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py -x -q -m gpu -k "big or tiny_teacher or config0 or long_sources" > gpurun_out/r2j/model.log 2>&1
python scripts/row_micro.py attn > gpurun_out/r2j/attn_generic.txt 2>&1
python scripts/row_micro.py src > gpurun_out/r2j/attn_tma.txt 2>&1
for i in 1 2; do
  MNMT_ATTN_TMA=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2j/bench_tma0_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2j/bench_tma1_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --smallm 32 --smallm-kmax 1024 > gpurun_out/r2j/bench_tma1_smallm_$i.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu > gpurun_out/r2j/parity.log 2>&1
cp gpurun_out/parity/r2_parity.jsonl gpurun_out/r2j/ 2>/dev/null
