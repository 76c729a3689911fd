#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the op-level kernel parity
# tests and one small model-level decode (tcgen05 / TMA / mbarrier GEMMs incl. split-K clusters,
# row kernels, attention, finish/compaction, PDL chains inside CUDA graphs).
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='gemm_acc_bitexact or split_k or gemm_epilogues or small_m or argmax or layernorm or aan_step or embed or attention or quantize or gather_rows'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
     python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "$SEL" -p no:cacheprovider \
     > gpurun_out/sanitize/$tool.kernels.log 2>&1
  echo "$tool kernels rc=$?" >> gpurun_out/sanitize/summary.txt
  tail -3 gpurun_out/sanitize/$tool.kernels.log >> gpurun_out/sanitize/summary.txt
  timeout 900 $CS --tool $tool $extra --target-processes all --print-limit 50 \
     python -m pytest tests/test_gpu_model.py -x -q -m gpu -k "tiny_teacher_forced and (t-aan or t-self) or config0" -p no:cacheprovider \
     > gpurun_out/sanitize/$tool.model.log 2>&1
  echo "$tool model rc=$?" >> gpurun_out/sanitize/summary.txt
  tail -3 gpurun_out/sanitize/$tool.model.log >> gpurun_out/sanitize/summary.txt
done
