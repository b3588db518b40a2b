#!/bin/bash
# full bench sweep (one JSON line per run) for DESIGN.md tables
mkdir -p gpurun_out/sweep
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/sweep/ours_$c.json 2> gpurun_out/sweep/ours_$c.err
done
for c in c3 c4; do
  timeout 900 python bench.py --config $c --mode global --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/global_$c.json 2> gpurun_out/sweep/global_$c.err
done
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --impl reference --config $c --steps 2 --warmup 0 > gpurun_out/sweep/ref_$c.json 2> gpurun_out/sweep/ref_$c.err
done
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/sweep/lscpu.txt
ls -la gpurun_out/sweep
