#!/bin/bash
# ncu --set full of the decoder's top kernels at the bench shape (one launch each, after warm-up)
mkdir -p gpurun_out/ncu
for k in dxd out attn attn16; do
  KERNEL=$k M=630 ncu --set full --clock-control none --import-source on -s 3 -c 1 -f \
      -o gpurun_out/ncu/$k python scripts/kernel_once.py > gpurun_out/ncu/$k.log 2>&1
  ncu -i gpurun_out/ncu/$k.ncu-rep --page raw --csv > gpurun_out/ncu/$k.csv 2>/dev/null
done
python scripts/ncu_full_summary.py \
  "dxd|M=630 N=256 K=256 (k_gemm_i8<32,EPI_F32>)|gpurun_out/ncu/dxd.csv" \
  "out|M=630 N=36000 K=256 (k_gemm_pers<256,EPI_ARGMAX>)|gpurun_out/ncu/out.csv" \
  "attn|rows=630 S=21 d=256 H=8 (k_attn, one layer)|gpurun_out/ncu/attn.csv" \
  "attn16|rows=630 S=21 d=256 H=8 (k_attn, bf16 K/V, one layer)|gpurun_out/ncu/attn16.csv" \
  > gpurun_out/ncu/summary.json
cat gpurun_out/ncu/summary.json
