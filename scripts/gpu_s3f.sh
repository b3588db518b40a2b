#!/bin/bash
# fused multi-class apply gather (PCB_FUSED_GATHER=1, default) vs one launch per class (=0)
mkdir -p gpurun_out
echo "== parity: $(timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_tools.py -q -x 2>&1 | tail -2)"
run() { # tag cfg env...
  tag=$1; cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3f_${cfg}_$tag.json 2>gpurun_out/s3f_${cfg}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/s3f_${cfg}_$tag.json'));print('$cfg $tag', round(d['value']), round(d['e2e']['value']), round(d['e2e'].get('registered_value',0)), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3f_${cfg}_$tag.err
}
for cfg in c3 c2 c1; do
run perclass $cfg PCB_FUSED_GATHER=0
run fused $cfg PCB_FUSED_GATHER=1
done
run fused_ml2 c3 PCB_FUSED_GATHER=1 PCB_MIXED_LAST=2
timeout 600 python scripts/hmatrix_time.py 2>&1 | grep -v "^{" | tail -6 | cut -c1-330
