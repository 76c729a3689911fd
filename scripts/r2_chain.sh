#!/bin/bash
mkdir -p gpurun_out/r2y
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SHAPES="8x256x256,128x256x256,8x1024x1024,32x1024x1024,128x1024x1024,630x1024x1024,8x3072x1024,8x4096x1024,8x1024x4096,128x1024x4096" python scripts/gemm_chain.py > gpurun_out/r2y/gemm_chain.txt 2>&1
for i in 1 2; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2y/bench_big_$i.json 2>/dev/null; done
