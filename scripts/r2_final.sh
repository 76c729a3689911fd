#!/bin/bash
# Final evidence of the current build: GPU tests, smoke, bench (default = big) with roofline and
# cpu_baseline, one-job launch list + decoder-GEMM pipe report, ncu --set full of the top kernels,
# other workloads' bench lines, the reference arm.
mkdir -p gpurun_out/fin/ncu
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin/gpu_tests.log 2>&1
cp gpurun_out/parity/r2_parity.jsonl gpurun_out/fin/ 2>/dev/null
python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
for w in small-aan-newstest-8192w base-aan-newstest-8192w base-newstest-8192w tiny192-aan-newstest-8192w; do
  python bench.py --workload $w --no-cpu-baseline > gpurun_out/fin/bench_$w.json 2>/dev/null
done
python bench.py --scaling strong --gpus 1 --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/fin/bench_strong1.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/bench_reference.json 2>/dev/null
PRESET=big OPTS="lanes=2,lane_tiers=15,pers_reserve=16,smallm=0,sab=64,attn_tma_self=2" timeout 1500 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active \
   --clock-control none --csv --log-file gpurun_out/fin/launches_big.csv python scripts/job_once.py > gpurun_out/fin/job_big.log 2>&1
python scripts/launch_summary.py gpurun_out/fin/launches_big.csv > gpurun_out/fin/launches_big_summary.txt
python scripts/gemm_pipe_report.py gpurun_out/fin/launches_big.csv --preset big --budget 8192 --mcr 4096 \
   --workload big-newstest-8192w --out gpurun_out/fin/decoder_gemm_pipe_big.md --json gpurun_out/fin/decoder_gemm_pipe_big.json
run() {
  local n=$1 k=$2; shift 2
  env "$@" timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -f \
      -o gpurun_out/fin/ncu/$n python scripts/kernel_once.py > gpurun_out/fin/ncu/$n.log 2>&1
  ncu -i gpurun_out/fin/ncu/$n.ncu-rep --page raw --csv > gpurun_out/fin/ncu/$n.csv 2>/dev/null
  ncu -i gpurun_out/fin/ncu/$n.ncu-rep --page details --print-details all > gpurun_out/fin/ncu/$n.details.txt 2>/dev/null
}
run sab_ffn2 'k_gemm' KERNEL=ffn2 D=1024 F=4096 M=32 NTILE=-2
run sab_dxd 'k_gemm' KERNEL=dxd D=1024 M=16 NTILE=-2
run enc_mq 'k_attn_enc' KERNEL=enc D=1024 H=16 M=2371 S=28 ENCV=2
run pair_ffn2 'k_gemm' KERNEL=ffn2 D=1024 F=4096 M=33000 NTILE=-3
run attn 'k_attn' KERNEL=attn D=1024 H=16 M=630 S=21
run ln 'k_ln' KERNEL=ln D=1024 M=630
run dxd 'k_gemm' KERNEL=dxd D=1024 M=630
run out 'k_gemm' KERNEL=out D=1024 M=630
python scripts/ncu_full_summary.py \
  "attn@big-newstest-8192w|rows=630 S=21 d=1024 H=16 (k_attn_tma, one layer)|gpurun_out/fin/ncu/attn.csv" \
  "ln@big-newstest-8192w|rows=630 d=1024 (k_ln_split<4>)|gpurun_out/fin/ncu/ln.csv" \
  "dxd@big-newstest-8192w|M=630 N=1024 K=1024 (k_gemm_i8<64,EPI_F32>)|gpurun_out/fin/ncu/dxd.csv" \
  "out@big-newstest-8192w|M=630 N=36000 K=1024 (k_gemm_pers<256,EPI_ARGMAX>)|gpurun_out/fin/ncu/out.csv" \
  "sab_ffn2@big-newstest-8192w|M=32 N=1024 K=4096 (k_gemm_sab<32,EPI_F32>, 4-CTA K split)|gpurun_out/fin/ncu/sab_ffn2.csv" \
  "sab_dxd@big-newstest-8192w|M=16 N=1024 K=1024 (k_gemm_sab<16,EPI_F32>)|gpurun_out/fin/ncu/sab_dxd.csv" \
  "enc_mq@big-newstest-8192w|2371 sentences of 10..28 tokens, d=1024 H=16 (k_attn_enc_mq<4>)|gpurun_out/fin/ncu/enc_mq.csv" \
  "pair_ffn2@big-newstest-8192w|M=33000 N=1024 K=4096 (k_gemm_pers2<EPI_F32>, CTA pairs)|gpurun_out/fin/ncu/pair_ffn2.csv" \
  > gpurun_out/fin/ncu_full_kernels.json
rm -f gpurun_out/fin/ncu/*.ncu-rep
