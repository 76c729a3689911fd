#!/bin/bash
# Full check of the current build: GPU tests, bench (default = big), one-job launch list and
# decoder-GEMM tensor-pipe report (big), ncu --set full of the top kernels at the bench shape.
mkdir -p gpurun_out/r2h/ncu
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2h/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2h/gpu_tests.log 2>&1
python bench.py > gpurun_out/r2h/bench.json 2> gpurun_out/r2h/bench.err
PRESET=big OPTS="lanes=3,lane_tiers=25,pers_reserve=16,smallm=0" timeout 1500 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active \
   --clock-control none --csv --log-file gpurun_out/r2h/launches_big.csv python scripts/job_once.py > gpurun_out/r2h/job_big.log 2>&1
python scripts/launch_summary.py gpurun_out/r2h/launches_big.csv > gpurun_out/r2h/launches_big_summary.txt
python scripts/gemm_pipe_report.py gpurun_out/r2h/launches_big.csv --preset big --budget 8192 --mcr 4096 \
   --workload big-newstest-8192w --out gpurun_out/r2h/decoder_gemm_pipe_big.md --json gpurun_out/r2h/decoder_gemm_pipe_big.json
run() {  # name, kernel regex, env...
  local n=$1 k=$2; shift 2
  env "$@" timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -f \
      -o gpurun_out/r2h/ncu/$n python scripts/kernel_once.py > gpurun_out/r2h/ncu/$n.log 2>&1
  ncu -i gpurun_out/r2h/ncu/$n.ncu-rep --page raw --csv > gpurun_out/r2h/ncu/$n.csv 2>/dev/null
}
run attn 'k_attn' KERNEL=attn D=1024 H=16 M=630 S=21
run ln 'k_ln' KERNEL=ln D=1024 M=630
run dxd 'k_gemm' KERNEL=dxd D=1024 M=630
run out 'k_gemm' KERNEL=out D=1024 M=630
run ffn2 'k_gemm' KERNEL=ffn2 D=1024 F=4096 M=32
python scripts/ncu_full_summary.py \
  "attn@big-newstest-8192w|rows=630 S=21 d=1024 H=16 (k_attn, one layer)|gpurun_out/r2h/ncu/attn.csv" \
  "ln@big-newstest-8192w|rows=630 d=1024 (k_ln_split<4>)|gpurun_out/r2h/ncu/ln.csv" \
  "dxd@big-newstest-8192w|M=630 N=1024 K=1024 (k_gemm_i8<64,EPI_F32>)|gpurun_out/r2h/ncu/dxd.csv" \
  "out@big-newstest-8192w|M=630 N=36000 K=1024 (k_gemm_pers<256,EPI_ARGMAX>)|gpurun_out/r2h/ncu/out.csv" \
  "ffn2@big-newstest-8192w|M=32 N=1024 K=4096 (split-K k_gemm_i8<64,EPI_F32>)|gpurun_out/r2h/ncu/ffn2.csv" \
  > gpurun_out/r2h/ncu_full_kernels.json
rm -f gpurun_out/r2h/ncu/*.ncu-rep
