#!/bin/bash
mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MNMT_SPLITK=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/r2e/kernels_splitk.log 2>&1
for v in 0 1; do MNMT_SPLITK=$v python scripts/gemm_micro.py 1024 4096 > gpurun_out/r2e/gemm_big_splitk$v.txt 2>&1; done
for v in 0 1; do MNMT_SPLITK=$v python scripts/gemm_micro.py 512 2048 > gpurun_out/r2e/gemm_base_splitk$v.txt 2>&1; done
for v in 0 1; do MNMT_SPLITK=$v PRESET=big BS=8,128,512 T=48 python scripts/step_latency.py lanes=1 > gpurun_out/r2e/step_big_splitk$v.txt 2>&1; done
MNMT_SPLITK=1 timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu -k "big" > gpurun_out/r2e/parity_big_splitk.log 2>&1
for v in 0 1; do MNMT_SPLITK=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2e/bench_big_splitk$v.json 2> gpurun_out/r2e/bench_big_splitk$v.err; done
