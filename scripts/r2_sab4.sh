#!/bin/bash
# big job: swap-AB bound / split-K cap / output-GEMM bound sweep; tier probe.
mkdir -p gpurun_out/sab4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sab4/build.log 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/sab4/$n.json 2>/dev/null; }
run def
run s64 --opt sab=64 --smallm 0
run s64_kb4 --opt sab=64 --smallm 0 --opt sab_kb=4
run s64_kb2 --opt sab=64 --smallm 0 --opt sab_kb=2
run s64_out16 --opt sab=64 --smallm 0 --opt sab_out=16
run s64_out8 --opt sab=64 --smallm 0 --opt sab_out=8
run s128 --opt sab=128 --smallm 0
run s64_kb4_sm --opt sab=64 --opt sab_kb=4
run s64_lanes3 --opt sab=64 --smallm 0 --lanes 3 --lane-tiers 25
run def_b
run s64_b --opt sab=64 --smallm 0
PRESET=big LANES=2 TIERS=15 GREEN=0 OPTS="smallm=0,sab=64,attn_tma_self=2" timeout 900 python scripts/tier_probe.py > gpurun_out/sab4/tier_probe_s64.txt 2>&1
