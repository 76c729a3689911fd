#!/bin/bash
mkdir -p gpurun_out/knobs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/knobs/build.log 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/knobs/$n.json 2>/dev/null; }
run small_def --workload small-aan-newstest-8192w
run small_sm0 --workload small-aan-newstest-8192w --smallm 0
run small_sab32 --workload small-aan-newstest-8192w --smallm 0 --sab 32
run baseaan_def --workload base-aan-newstest-8192w
run baseaan_sm0 --workload base-aan-newstest-8192w --smallm 0
run baseaan_sab32 --workload base-aan-newstest-8192w --smallm 0 --sab 32
run base_sab32 --workload base-newstest-8192w --sab 32
run base_def --workload base-newstest-8192w
run big_def
run big_splitk --opt split_k=1
run tiny_sab32 --workload tiny192-aan-newstest-8192w --sab 32
run tiny_def --workload tiny192-aan-newstest-8192w
