#!/bin/bash
# cols L2 experiments: family-ordered slots (PCB_SLOT_FAM=1), streaming T stores (build/ab/tcs.so)
mkdir -p gpurun_out
echo "== parity (PCB_SLOT_FAM=1): $(PCB_SLOT_FAM=1 timeout 900 python -m pytest tests/test_gpu_headline.py -q -x -k 'fingerprint' 2>&1 | tail -1)"
run() { # tag cfg env...
  tag=$1; cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3e_${cfg}_$tag.json 2>gpurun_out/s3e_${cfg}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/s3e_${cfg}_$tag.json'));print('$cfg $tag', round(d['value']), round(d['e2e']['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3e_${cfg}_$tag.err
}
for cfg in c3 c4 c2; do
run base $cfg A=1
run slotfam $cfg PCB_SLOT_FAM=1
run tcs $cfg PCB_LIB_PATH=$PWD/build/ab/tcs.so
run tcs_slotfam $cfg PCB_LIB_PATH=$PWD/build/ab/tcs.so PCB_SLOT_FAM=1
done
