#!/bin/bash
mkdir -p gpurun_out/tiers
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/tiers/$n.json 2>/dev/null; }
for t in 15 12 13 17 18 15; do run big_t$t --lane-tiers $t; done
