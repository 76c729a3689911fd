#!/bin/bash
mkdir -p gpurun_out/outtile
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "argmax or gemm_acc or epilogues" > gpurun_out/outtile/tests.log 2>&1
echo "rc=$?" >> gpurun_out/outtile/tests.log
timeout 300 python scripts/out_micro.py 1024 > gpurun_out/outtile/out_1024.txt 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/outtile/$n.json 2>/dev/null; }
for i in a b; do
run big_$i
run small_$i --workload small-aan-newstest-8192w
run baseaan_$i --workload base-aan-newstest-8192w
run base_$i --workload base-newstest-8192w
run tiny_$i --workload tiny192-aan-newstest-8192w
done
