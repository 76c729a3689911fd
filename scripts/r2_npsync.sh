#!/bin/bash
mkdir -p gpurun_out/npsync
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/npsync/build.log 2>&1
for v in 0 1; do
  MNMT_NPSYNC=$v MNMT_GEMM_PERSISTENT=0 timeout 600 python scripts/gemm_micro.py 1024 4096 > gpurun_out/npsync/micro_big_np_s$v.txt 2>&1
  MNMT_NPSYNC=$v timeout 600 python scripts/gemm_micro.py 256 2048 > gpurun_out/npsync/micro_small_s$v.txt 2>&1
done
MNMT_NPSYNC=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/npsync/tests.log 2>&1
echo "rc=$?" >> gpurun_out/npsync/tests.log
