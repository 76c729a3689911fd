#!/bin/bash
# d_h = 64 multi-query encoder attention: parity, ncu --set full (generic vs QW = 4 / 8), job A/B;
# swap-AB micro with one accumulator (conditional TMEM allocation).
mkdir -p gpurun_out/enc/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/enc/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swap_ab or attention_enc" > gpurun_out/enc/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/enc/tests.log
ROWS=1,16,64 timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/enc/micro_big.txt 2>&1
for v in 1 2 3; do
  KERNEL=enc M=2371 S=28 D=1024 H=16 ENCV=$v timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_attn_enc -s 3 -c 1 -f \
      -o gpurun_out/enc/ncu/enc_v$v python scripts/kernel_once.py > gpurun_out/enc/ncu/enc_v$v.log 2>&1
  ncu -i gpurun_out/enc/ncu/enc_v$v.ncu-rep --page raw --csv > gpurun_out/enc/ncu/enc_v$v.csv 2>/dev/null
  ncu -i gpurun_out/enc/ncu/enc_v$v.ncu-rep --page details --print-details all > gpurun_out/enc/ncu/enc_v$v.details.txt 2>/dev/null
  ncu -i gpurun_out/enc/ncu/enc_v$v.ncu-rep --page source --csv > gpurun_out/enc/ncu/enc_v$v.source.csv 2>/dev/null
done
rm -f gpurun_out/enc/ncu/*.ncu-rep
for mq in 0 4 8; do
  MNMT_ENC_MQ=$mq timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/enc/big_mq$mq.json 2>/dev/null
done
MNMT_ENC_MQ=4 timeout 600 python bench.py --workload base-aan-newstest-8192w --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/enc/baseaan_mq4.json 2>/dev/null
MNMT_ENC_MQ=0 timeout 600 python bench.py --workload base-aan-newstest-8192w --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/enc/baseaan_mq0.json 2>/dev/null
