#!/bin/bash
mkdir -p gpurun_out/bpre
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bpre/build.log 2>&1
for v in -1 0 1 2; do MNMT_BPRE=$v timeout 600 python scripts/gemm_micro.py 1024 4096 > gpurun_out/bpre/micro_big_b$v.txt 2>&1; done
MNMT_BPRE=0 timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/bpre/micro_small_b0.txt 2>&1
MNMT_BPRE=0 MNMT_GEMM_PERSISTENT=1 timeout 600 python scripts/gemm_micro.py 1024 4096 > gpurun_out/bpre/micro_big_b0_p1.txt 2>&1
MNMT_BPRE=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/bpre/tests.log 2>&1
echo "rc=$?" >> gpurun_out/bpre/tests.log
