#!/bin/bash
# round 2 (c): reference H-matrix parity, VB sweep (L2 residency of S/T), ncu of the apply cols, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hmatrix_ref.py tests/test_gpu_hmatrix.py -q -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_c.log
for vb in 1 2 4 8 16 64; do
  PCB_VB=$vb timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/vb_$vb.json 2> gpurun_out/vb_$vb.err
  python -c "import json;d=json.load(open('gpurun_out/vb_$vb.json'));print('VB=$vb', round(d['value']), round(d['ms_per_step'],3), d['kernels_ms_per_step'])" || tail -3 gpurun_out/vb_$vb.err
done
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cols -s 15 -c 1 -o gpurun_out/r02c_c3_cols $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_c.json 2> gpurun_out/bench_c3_c.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_c3_c.json'));print(d['value'], d['e2e'], d['roofline'])"
