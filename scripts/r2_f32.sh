#!/bin/bash
mkdir -p gpurun_out/f32
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f32/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm or attention" > gpurun_out/f32/tests.log 2>&1
echo "kernel tests rc=$?" >> gpurun_out/f32/tests.log
timeout 1800 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "attn_f32" >> gpurun_out/f32/tests.log 2>&1
echo "f32 model tests rc=$?" >> gpurun_out/f32/tests.log
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/f32/$n.json 2>/dev/null; }
run big_def
run big_f32 --opt attn_f32=1
run base_def --workload base-newstest-8192w
run base_f32 --workload base-newstest-8192w --opt attn_f32=1
run baseaan_def --workload base-aan-newstest-8192w
run small_def --workload small-aan-newstest-8192w
run big_def_b
