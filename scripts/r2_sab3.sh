#!/bin/bash
# swap-AB argmax with a CTA-level row maximum; sab row bound on every workload.
mkdir -p gpurun_out/sab3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sab3/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swap_ab or argmax" > gpurun_out/sab3/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/sab3/tests.log
ROWS=1,8,16,32,64 timeout 600 python scripts/sab_micro.py 1024 4096 2>&1 | grep "^out" > gpurun_out/sab3/micro_out.txt
ROWS=1,8,16,32 timeout 600 python scripts/sab_micro.py 256 2048 > gpurun_out/sab3/micro_small.txt 2>&1
ROWS=1,8,16,32 timeout 600 python scripts/sab_micro.py 512 2048 > gpurun_out/sab3/micro_base.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/sab3/$n.json 2>/dev/null; }
run big_def
run big_sab32 --opt sab=32
run big_sab16 --opt sab=16
run big_sab64 --opt sab=64
run big_sab32_nosmallm --opt sab=32 --smallm 0
for w in small-aan base-aan base tiny192-aan; do
  run ${w}_def --workload $w-newstest-8192w
  run ${w}_sab32 --workload $w-newstest-8192w --opt sab=32
  run ${w}_sab16 --workload $w-newstest-8192w --opt sab=16
done
run big_sab32_b --opt sab=32
run big_def_b
