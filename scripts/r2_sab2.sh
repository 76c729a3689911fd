#!/bin/bash
# Swap-AB epilogue (staged stores, redux argmax) + live-row A boxes / 32-row B boxes in k_gemm_i8:
# op-level parity, warm micro A/B, whole-job A/B.
mkdir -p gpurun_out/sab2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sab2/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/sab2/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/sab2/tests.log
timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/sab2/micro_big.txt 2>&1
MNMT_ABOX=0 ROWS=1,16,32,64 timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/sab2/micro_big_noabox.txt 2>&1
timeout 600 python scripts/sab_micro.py 256 2048 > gpurun_out/sab2/micro_small.txt 2>&1
for s in 0 32 64; do
  timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline --opt sab=$s > gpurun_out/sab2/big_sab$s.json 2> gpurun_out/sab2/big_sab$s.err
done
MNMT_ABOX=0 timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/sab2/big_noabox.json 2>/dev/null
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline --smallm 0 --opt sab=32 > gpurun_out/sab2/big_sab32_nosmallm.json 2>/dev/null
for w in small-aan-newstest-8192w base-aan-newstest-8192w; do
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/sab2/${w}_def.json 2>/dev/null
  MNMT_ABOX=0 timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/sab2/${w}_noabox.json 2>/dev/null
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-roofline --opt sab=32 > gpurun_out/sab2/${w}_sab32.json 2>/dev/null
done
