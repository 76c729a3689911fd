#!/bin/bash
# Independent TMEM accumulators (MNMT_NACC) in the swap-AB kernel; d_h = 64 multi-query encoder
# attention (MNMT_ENC_MQ) tests and job A/B.
mkdir -p gpurun_out/nacc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/nacc/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swap_ab or attention_enc" > gpurun_out/nacc/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/nacc/tests.log
MNMT_NACC=4 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swap_ab" >> gpurun_out/nacc/tests.log 2>&1
echo "tests nacc4 rc=$?" >> gpurun_out/nacc/tests.log
for n in 1 2 4; do
  MNMT_NACC=$n ROWS=1,16,64 timeout 600 python scripts/sab_micro.py 1024 4096 > gpurun_out/nacc/micro_big_nacc$n.txt 2>&1
done
for mq in 0 4 8; do
  MNMT_ENC_MQ=$mq timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/nacc/big_mq$mq.json 2>/dev/null
  MNMT_ENC_MQ=$mq timeout 600 python bench.py --workload small-aan-newstest-8192w --steps 5 --no-cpu-baseline --no-roofline > gpurun_out/nacc/small_mq$mq.json 2>/dev/null
done
MNMT_ENC_MQ=0 PRESET=big OPTS="lanes=2,lane_tiers=15,pers_reserve=16,smallm=32,smallm_kmax=1024,attn_tma_self=2" timeout 900 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_attn_enc --log-file gpurun_out/nacc/enc_mq0.csv python scripts/job_once.py > /dev/null 2>&1
MNMT_ENC_MQ=4 PRESET=big OPTS="lanes=2,lane_tiers=15,pers_reserve=16,smallm=32,smallm_kmax=1024,attn_tma_self=2" timeout 900 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_attn_enc --log-file gpurun_out/nacc/enc_mq4.csv python scripts/job_once.py > /dev/null 2>&1
MNMT_ENC_MQ=8 PRESET=big OPTS="lanes=2,lane_tiers=15,pers_reserve=16,smallm=32,smallm_kmax=1024,attn_tma_self=2" timeout 900 ncu --nvtx --nvtx-include "job/" \
   --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_attn_enc --log-file gpurun_out/nacc/enc_mq8.csv python scripts/job_once.py > /dev/null 2>&1
