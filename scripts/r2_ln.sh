#!/bin/bash
mkdir -p gpurun_out/r2d
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MNMT_LN_SPLIT=0 python scripts/row_micro.py ln > gpurun_out/r2d/ln_warp.txt 2>&1
python scripts/row_micro.py ln > gpurun_out/r2d/ln_split.txt 2>&1
python scripts/row_micro.py attn > gpurun_out/r2d/attn.txt 2>&1
for v in 0 1; do MNMT_LN_SPLIT=$v PRESET=big BS=8,128,512,2048 T=48 python scripts/step_latency.py lanes=1 > gpurun_out/r2d/step_big_split$v.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/r2d/tests_quick.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu -v > gpurun_out/r2d/parity.log 2>&1
cp gpurun_out/parity/r2_parity.jsonl gpurun_out/r2d/ 2>/dev/null
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2d/bench_big.json 2> gpurun_out/r2d/bench_big.err
