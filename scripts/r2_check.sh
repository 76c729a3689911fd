#!/bin/bash
# Refactor check: GPU test suite + ncu --set full of the big student's top kernels.
mkdir -p gpurun_out/r2c/ncu
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2c/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2c/gpu_tests.log 2>&1
run() {  # name, env...
  local n=$1; shift
  env "$@" timeout 300 ncu --set full --clock-control none --import-source on -s 3 -c 1 -f \
      -o gpurun_out/r2c/ncu/$n python scripts/kernel_once.py > gpurun_out/r2c/ncu/$n.log 2>&1
  ncu -i gpurun_out/r2c/ncu/$n.ncu-rep --page raw --csv > gpurun_out/r2c/ncu/$n.csv 2>/dev/null
  ncu -i gpurun_out/r2c/ncu/$n.ncu-rep --page details --csv > gpurun_out/r2c/ncu/$n.details.csv 2>/dev/null
}
run ln_big KERNEL=ln D=1024 M=256
run ln_small KERNEL=ln D=256 M=256
run attn_big KERNEL=attn D=1024 H=16 M=512 S=21
run dxd_big KERNEL=dxd D=1024 M=128
run ffn1_big KERNEL=ffn1 D=1024 F=4096 M=128
rm -f gpurun_out/r2c/ncu/*.ncu-rep.tmp
