#!/bin/bash
# compute-sanitizer over the round-2b kernels: swap-AB GEMM (split-K clusters, staged epilogue,
# CTA argmax), live-row A boxes in k_gemm_i8, multi-query encoder attention.
mkdir -p gpurun_out/sanitize_sab
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='swap_ab or attention_enc or gemm_epilogues or split_k'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 30 \
     python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "$SEL" -p no:cacheprovider \
     > gpurun_out/sanitize_sab/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_sab/summary.txt
  tail -3 gpurun_out/sanitize_sab/$tool.log >> gpurun_out/sanitize_sab/summary.txt
done
