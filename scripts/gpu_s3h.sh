#!/bin/bash
# knob re-sweep on the final kernels: row-pass occupancy targets, bundle members per round, CTA size
mkdir -p gpurun_out
run() { tag=$1; shift
  env "$@" python bench.py --config c3 --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3h_$tag.json 2>gpurun_out/s3h_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/s3h_$tag.json'));print('c3 $tag', round(d['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3h_$tag.err
}
run base A=1
for lib in build/ab/*.so; do run $(basename $lib .so) PCB_LIB_PATH=$PWD/$lib; done
run base2 A=1
