#!/bin/bash
# A/B of the GLOBAL plan (c3, c4) between the in-tree library and build/ab/*.so variants
mkdir -p gpurun_out
for cfg in ${CFGS:-c3 c4}; do
  for lib in default build/ab/*.so; do
    if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
    tag=$(basename $lib .so)
    python bench.py --config $cfg --mode global --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abg_${cfg}_$tag.json 2> gpurun_out/abg_${cfg}_$tag.err
    python -c "import json;d=json.load(open('gpurun_out/abg_${cfg}_$tag.json'));r=d['roofline'];print('$cfg $tag', round(d['value'],1), r['kernel'], round(r['frac'],3), round(r['fp64']['frac'],3), {k: round(v,2) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/abg_${cfg}_$tag.err
  done
done
unset PCB_LIB_PATH
