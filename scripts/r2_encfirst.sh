#!/bin/bash
# enc_first scheduling A/B on every workload; compute-sanitizer over the new kernels.
mkdir -p gpurun_out/encfirst
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/encfirst/build.log 2>&1
run() { local n=$1; shift; timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-roofline "$@" > gpurun_out/encfirst/$n.json 2>/dev/null; }
run big_def
run big_ef --opt enc_first=1
for w in small-aan base-aan base tiny192-aan; do
  run ${w}_def --workload $w-newstest-8192w
  run ${w}_ef --workload $w-newstest-8192w --opt enc_first=1
done
run big_ef_b --opt enc_first=1
run big_def_b
bash scripts/sanitize_sab.sh
