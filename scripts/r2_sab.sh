#!/bin/bash
# Swap-AB GEMM: op-level parity, warm micro A/B against the 128-row tcgen05 and IDP4A kernels,
# whole-job A/B of the sab row bound on the big / small-AAN / base-AAN jobs.
mkdir -p gpurun_out/sab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sab/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swap_ab or gemm" > gpurun_out/sab/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/sab/tests.log
timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/sab/micro_big.txt 2>&1
timeout 600 python scripts/sab_micro.py 256 2048 > gpurun_out/sab/micro_small.txt 2>&1
for s in 0 32 64 128; do
  timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline --opt sab=$s > gpurun_out/sab/big_sab$s.json 2> gpurun_out/sab/big_sab$s.err
done
for s in 0 64; do
  timeout 600 python bench.py --workload small-aan-newstest-8192w --steps 5 --no-cpu-baseline --no-roofline --opt sab=$s > gpurun_out/sab/small_sab$s.json 2>/dev/null
  timeout 600 python bench.py --workload base-aan-newstest-8192w --steps 5 --no-cpu-baseline --no-roofline --opt sab=$s > gpurun_out/sab/baseaan_sab$s.json 2>/dev/null
done
