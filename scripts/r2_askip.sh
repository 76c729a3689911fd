#!/bin/bash
mkdir -p gpurun_out/r2x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -m gpu > gpurun_out/r2x/tests.log 2>&1
python scripts/gemm_micro.py 1024 4096 > gpurun_out/r2x/gemm_big.txt 2>&1
b() { local tag=$1; shift; env $ENVV python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline "$@" > gpurun_out/r2x/bench_$tag.json 2>/dev/null; }
for i in 1 2; do
ENVV="MNMT_A_SKIP=0" b noskip_$i
ENVV="" b skip_$i
ENVV="" b skip_smallm_$i --smallm 32 --smallm-kmax 1024
ENVV="" b skip_t10_$i --lane-tiers 10
done
for w in small-aan-newstest-8192w base-aan-newstest-8192w base-newstest-8192w tiny192-aan-newstest-8192w; do
  ENVV="MNMT_A_SKIP=0" b ${w}_noskip --workload $w
  ENVV="" b ${w}_skip --workload $w
done
