#!/bin/bash
mkdir -p gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -m gpu > gpurun_out/r2k/tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu > gpurun_out/r2k/parity.log 2>&1
cp gpurun_out/parity/r2_parity.jsonl gpurun_out/r2k/ 2>/dev/null
for i in 1 2; do
  MNMT_ENC_R64=0 MNMT_ATTN_TMA=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2k/bench_old_$i.json 2>/dev/null
  MNMT_ENC_R64=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2k/bench_tma_$i.json 2>/dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2k/bench_tma_enc_$i.json 2>/dev/null
done
for w in base-newstest-8192w base-aan-newstest-8192w small-aan-newstest-8192w; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/r2k/bench_$w.json 2>/dev/null
done
PRESET=big GREEN=0 TIERS=25 python scripts/tier_probe.py > gpurun_out/r2k/tier_probe_big.txt 2>&1
