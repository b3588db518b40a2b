#!/bin/bash
# A/B: bench.py with the in-tree library vs alternative builds under build/ab/*.so
# usage: CFGS="c3 c4" bash scripts/ab_bench.sh
mkdir -p gpurun_out
for cfg in ${CFGS:-c3}; do
  for lib in default build/ab/*.so; do
    if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
    tag=$(basename $lib .so)
    python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${cfg}_$tag.json 2> gpurun_out/ab_${cfg}_$tag.err
    python - <<PY
import json
d = json.load(open("gpurun_out/ab_${cfg}_$tag.json"))
r = d["roofline"]
print("$cfg", "$tag", round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"], 3), r["kernel"], round(r["kernel_ms_per_step"], 3), round(r["frac"], 3), {k: round(v, 3) for k, v in d["kernels_ms_per_step"].items()})
PY
  done
done
unset PCB_LIB_PATH
