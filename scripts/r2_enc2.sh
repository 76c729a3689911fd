#!/bin/bash
# mq encoder attention without bank conflicts; swap-AB row / K bounds on the big job.
mkdir -p gpurun_out/enc2/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/enc2/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/enc2/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/enc2/tests.log
ROWS=1,16,32,64 timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/enc2/micro_big.txt 2>&1
for v in 2 3; do
  KERNEL=enc M=2371 S=28 D=1024 H=16 ENCV=$v timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_attn_enc -s 3 -c 1 -f \
      -o gpurun_out/enc2/ncu/enc_v$v python scripts/kernel_once.py > gpurun_out/enc2/ncu/enc_v$v.log 2>&1
  ncu -i gpurun_out/enc2/ncu/enc_v$v.ncu-rep --page raw --csv > gpurun_out/enc2/ncu/enc_v$v.csv 2>/dev/null
  ncu -i gpurun_out/enc2/ncu/enc_v$v.ncu-rep --page details --print-details all > gpurun_out/enc2/ncu/enc_v$v.details.txt 2>/dev/null
done
rm -f gpurun_out/enc2/ncu/*.ncu-rep
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/enc2/$n.json 2>/dev/null; }
run big_def
MNMT_ENC_MQ=0 run big_mq0
run big_sab32_k2048 --opt sab=32 --opt sab_kmin=2048
run big_sab64_k2048 --opt sab=64 --opt sab_kmin=2048
run big_sab32_k0 --opt sab=32
run big_def2
MNMT_ENC_MQ=8 run big_mq8
