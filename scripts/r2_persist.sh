#!/bin/bash
mkdir -p gpurun_out/persist
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/persist/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > gpurun_out/persist/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/persist/tests.log
timeout 600 python scripts/attn_persist_micro.py 1024 16 > gpurun_out/persist/micro_big.txt 2>&1
timeout 600 python scripts/attn_persist_micro.py 512 8 > gpurun_out/persist/micro_base.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/persist/$n.json 2>/dev/null; }
run big_def
run big_p1 --opt attn_persist=1
run baseaan_def --workload base-aan-newstest-8192w
run baseaan_p1 --workload base-aan-newstest-8192w --opt attn_persist=1
run small_def --workload small-aan-newstest-8192w
run small_p1 --workload small-aan-newstest-8192w --opt attn_persist=1
run big_p1_b --opt attn_persist=1
run big_def_b
