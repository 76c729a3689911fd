#!/bin/bash
mkdir -p gpurun_out/ncuattn
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() {
  local n=$1 k=$2; shift 2
  env "$@" timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -f \
      -o gpurun_out/ncuattn/$n python scripts/kernel_once.py > gpurun_out/ncuattn/$n.log 2>&1
  ncu -i gpurun_out/ncuattn/$n.ncu-rep --page details --print-details all > gpurun_out/ncuattn/$n.details.txt 2>/dev/null
  ncu -i gpurun_out/ncuattn/$n.ncu-rep --page source --csv --print-source sass > gpurun_out/ncuattn/$n.sass.csv 2>/dev/null
  ncu -i gpurun_out/ncuattn/$n.ncu-rep --page source --csv > gpurun_out/ncuattn/$n.src.csv 2>/dev/null
}
run split 'k_attn' KERNEL=attn D=1024 H=16 M=32 S=80
run one 'k_attn' KERNEL=attn D=1024 H=16 M=630 S=21
rm -f gpurun_out/ncuattn/*.ncu-rep
