#!/bin/bash
mkdir -p gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MNMT_ATTN_FAST=0 python scripts/row_micro.py attn > gpurun_out/r2g/attn_generic.txt 2>&1
MNMT_ATTN_MINB=2 python scripts/row_micro.py attn > gpurun_out/r2g/attn_fast2.txt 2>&1
MNMT_ATTN_MINB=1 python scripts/row_micro.py attn > gpurun_out/r2g/attn_fast1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/r2g/kernels.log 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py -x -q -m gpu -k "teacher_forced or long_sources or config0" > gpurun_out/r2g/model.log 2>&1
for v in 1 2; do MNMT_ATTN_MINB=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2g/bench_big_minb$v.json 2> gpurun_out/r2g/bench_big_minb$v.err; done
MNMT_ATTN_FAST=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2g/bench_big_generic.json 2> gpurun_out/r2g/bench_big_generic.err
