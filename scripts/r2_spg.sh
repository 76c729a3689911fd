#!/bin/bash
mkdir -p gpurun_out/spg
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/spg/$n.json 2>/dev/null; }
run big_1
run big_2 --steps-per-graph 2
run big_4 --steps-per-graph 4
run small_1 --workload small-aan-newstest-8192w
run small_2 --workload small-aan-newstest-8192w --steps-per-graph 2
run small_4 --workload small-aan-newstest-8192w --steps-per-graph 4
run big_2b --steps-per-graph 2
run big_1b
