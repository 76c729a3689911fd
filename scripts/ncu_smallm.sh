#!/bin/bash
# ncu --set full of one d x d decoder GEMM at 8 and 32 live rows: small-M IDP4A kernel vs the
# tcgen05 kernel (same shape), plus CUDA-event timing of both in a PDL chain is in step_latency.
mkdir -p gpurun_out/ncu_sm
for m in 8 32; do
  for nt in -1 0; do
    tag=m${m}_nt${nt}
    KERNEL=dxd M=$m NTILE=$nt ncu --set full --clock-control none --import-source on -s 3 -c 1 -f \
        -o gpurun_out/ncu_sm/$tag python scripts/kernel_once.py > gpurun_out/ncu_sm/$tag.log 2>&1
    ncu -i gpurun_out/ncu_sm/$tag.ncu-rep --page raw --csv > gpurun_out/ncu_sm/$tag.csv 2>/dev/null
  done
done
python scripts/ncu_full_summary.py \
  "smallm_m8|M=8 N=256 K=256 (k_gemm_smallm<EPI_F32,4,4>)|gpurun_out/ncu_sm/m8_nt-1.csv" \
  "tc_m8|M=8 N=256 K=256 (k_gemm_i8<32,EPI_F32>)|gpurun_out/ncu_sm/m8_nt0.csv" \
  "smallm_m32|M=32 N=256 K=256 (k_gemm_smallm<EPI_F32,4,4>)|gpurun_out/ncu_sm/m32_nt-1.csv" \
  "tc_m32|M=32 N=256 K=256 (k_gemm_i8<32,EPI_F32>)|gpurun_out/ncu_sm/m32_nt0.csv" \
  > gpurun_out/ncu_sm/summary.json
cat gpurun_out/ncu_sm/summary.json
