#!/bin/bash
mkdir -p gpurun_out/tconly
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/tconly/$n.json 2>/dev/null; }
for i in a b; do
W=small-aan-newstest-8192w
run small_def_$i --workload $W
run small_tc32_$i --workload $W --smallm 0 --sab 32
run small_tc32o_$i --workload $W --smallm 0 --sab 32 --opt sab_out=32
W=base-aan-newstest-8192w
run baseaan_def_$i --workload $W
run baseaan_tc32_$i --workload $W --smallm 0 --sab 32
run baseaan_tc64_$i --workload $W --smallm 0 --sab 64
done
