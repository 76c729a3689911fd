#!/bin/bash
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MNMT_SPLITK=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "gemm" > gpurun_out/r2f/kernels_splitk.log 2>&1
MNMT_SPLITK=1 python scripts/gemm_micro.py 1024 4096 > gpurun_out/r2f/gemm_big_splitk1.txt 2>&1
MNMT_SPLITK=1 MNMT_SPLITK_KMIN=512 python scripts/gemm_micro.py 512 2048 > gpurun_out/r2f/gemm_base_splitk1.txt 2>&1
MNMT_SPLITK=1 PRESET=big BS=8,128,512 T=48 python scripts/step_latency.py lanes=1 > gpurun_out/r2f/step_big_splitk1.txt 2>&1
