#!/bin/bash
mkdir -p gpurun_out/r2w
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { local tag=$1; shift; env $ENVV python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline "$@" > gpurun_out/r2w/bench_$tag.json 2>/dev/null; }
ENVV="" b l2_t25 --lanes 2
ENVV="" b l2_t15 --lanes 2 --lane-tiers 15
ENVV="" b l2_t35 --lanes 2 --lane-tiers 35
ENVV="" b l3_t15 --lanes 3 --lane-tiers 15
ENVV="" b l3_t10 --lanes 3 --lane-tiers 10
ENVV="MNMT_BN32_KMAX=1024" b l3_t25_bn32
ENVV="MNMT_BN32_KMAX=1024" b l2_t25_bn32 --lanes 2
ENVV="" b l3_t25_smallm --smallm 32 --smallm-kmax 1024
ENVV="" b l2_t25_smallm --lanes 2 --smallm 32 --smallm-kmax 1024
ENVV="" b l2_t25_r0 --lanes 2 --pers-reserve 0
ENVV="" b l2_t25_r32 --lanes 2 --pers-reserve 32
ENVV="" b l3_t25 
