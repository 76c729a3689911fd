#!/bin/bash
mkdir -p gpurun_out/r2p
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KERNEL=attn D=1024 H=16 M=630 S=21 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_attn" -s 3 -c 1 -f \
   -o gpurun_out/r2p/attn_tma python scripts/kernel_once.py > gpurun_out/r2p/attn_tma.log 2>&1
ncu -i gpurun_out/r2p/attn_tma.ncu-rep --page raw --csv > gpurun_out/r2p/attn_tma.csv 2>/dev/null
ncu -i gpurun_out/r2p/attn_tma.ncu-rep --page details --print-details all > gpurun_out/r2p/attn_tma_details.txt 2>/dev/null
ncu -i gpurun_out/r2p/attn_tma.ncu-rep --page source --csv --print-source sass > gpurun_out/r2p/attn_tma_sass.csv 2>/dev/null
python scripts/ncu_full_summary.py "attn@big-newstest-8192w|rows=630 S=21 d=1024 H=16 (k_attn_tma, one layer)|gpurun_out/r2p/attn_tma.csv" > gpurun_out/r2p/attn_summary.json
