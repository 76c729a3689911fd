#!/bin/bash
mkdir -p gpurun_out/green
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/green/$n.json 2>/dev/null; }
run big_g0
run big_g64 --green-sms 64
run big_g96 --green-sms 96
run big_g120 --green-sms 120
run big_l3g64 --lanes 3 --lane-tiers 15 --green-sms 64
run big_g0b
