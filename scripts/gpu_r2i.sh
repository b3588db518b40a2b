#!/bin/bash
# round 2 (i): c5 (classify with TMA zero stores + gather kernel); 3-smooth R2C rows with 12-element engines (A/B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_tools.py -q -p no:cacheprovider -k "c5 or blocks or guard" > gpurun_out/pytest_i.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_i.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; head -6 gpurun_out/c5_time.json
python scripts/c5_time.py > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python scripts/c5_time.py > /dev/null 2>&1; echo "ncu rc=$?"
for lib in default build/ab/rows12_96.so build/ab/rows12_192.so; do
  for ml in 0 1; do
    if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
    PCB_MIXED_LAST=$ml python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abm.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abm.json'));print('$lib ML=$ml', round(d['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done
unset PCB_LIB_PATH
