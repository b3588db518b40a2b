#!/bin/bash
# bundled gather: member descriptors staged in shared memory (default) vs loaded per round (build/ab/sdesc0.so)
mkdir -p gpurun_out
echo "== parity: $(timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -q -x -k 'fingerprint or bundled or split3 or families or vs_oracle or golden' 2>&1 | tail -1)"
run() { tag=$1; cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3j_${cfg}_$tag.json 2>gpurun_out/s3j_${cfg}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/s3j_${cfg}_$tag.json'));print('$cfg $tag', round(d['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3j_${cfg}_$tag.err
}
for cfg in c3 c2 c1; do
run sdesc1 $cfg A=1
run sdesc0 $cfg PCB_LIB_PATH=$PWD/build/ab/sdesc0.so
done
python scripts/adjoint_time.py 2>/dev/null | tail -1 | cut -c1-400
