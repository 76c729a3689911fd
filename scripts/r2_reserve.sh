#!/bin/bash
mkdir -p gpurun_out/reserve
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/reserve/$n.json 2>/dev/null; }
for r in 16 0 32 48 64; do run big_r$r --pers-reserve $r; done
run big_r16b --pers-reserve 16
for r in 16 32 48; do run small_r$r --workload small-aan-newstest-8192w --pers-reserve $r; done
for r in 16 32 48; do run baseaan_r$r --workload base-aan-newstest-8192w --pers-reserve $r; done
