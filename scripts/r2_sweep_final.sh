#!/bin/bash
mkdir -p gpurun_out/swf
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/swf/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" > gpurun_out/swf/tests.log 2>&1
echo "rc=$?" >> gpurun_out/swf/tests.log
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/swf/$n.json 2>/dev/null; }
run big_s64
run big_s32 --sab 32
run big_s16 --sab 16
run big_s32_o16 --sab 32 --opt sab_out=16
W=small-aan-newstest-8192w
run small_def --workload $W
run small_o32 --workload $W --sab 32 --opt sab_out=32
run small_k512_o32 --workload $W --smallm-kmax 512 --sab 32 --opt sab_out=32
W=base-aan-newstest-8192w
run baseaan_def --workload $W
run baseaan_o32 --workload $W --sab 32 --opt sab_out=32
W=base-newstest-8192w
run base_def --workload $W
run base_o32 --workload $W --sab 32 --opt sab_out=32
W=tiny192-aan-newstest-8192w
run tiny_def --workload $W
run tiny_o32 --workload $W --sab 32 --opt sab_out=32
run tiny_sm32_o32 --workload $W --smallm 32 --sab 32 --opt sab_out=32
run big_s64_b
