#!/bin/bash
# c5 blocks: one launch (union-box zero test, gather CTAs + zero-fill CTAs; mode 5) vs the classify + gather passes (mode 0)
mkdir -p gpurun_out
echo "== tests: $(timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_tools.py tests/test_gpu_hmatrix_ref.py -q -x -k 'c5 or block or guard or hmatrix' 2>&1 | tail -2)"
run() { # label env...
  env "$@" python scripts/c5_time.py > gpurun_out/s3d_c5.json 2> gpurun_out/s3d_c5.err
  python -c "import json;d=json.load(open('gpurun_out/s3d_c5.json'));print('$*: us/call %.1f kernel %.1f frac %.3f'%(d['ms_per_call']*1e3,d['kernel_ms']*1e3,d['frac_hbm']), {k: round(v*1e3,1) for k,v in d['split_ms'].items()})" || tail -3 gpurun_out/s3d_c5.err
}
run PCB_C5_ZERO=5
run PCB_C5_ZERO=5 PCB_C5_ZCTAS=1
run PCB_C5_ZERO=5 PCB_C5_ZCTAS=2
run PCB_C5_ZERO=5 PCB_C5_ZCTAS=3
run PCB_C5_ZERO=6 PCB_C5_ZCTAS=2
export PCB_LIB_PATH=$PWD/build/ab/bz4096.so
run PCB_C5_ZERO=5
run PCB_C5_ZERO=6
run PCB_C5_ZERO=5 PCB_C5_ZCTAS=1
run PCB_C5_ZERO=5 PCB_C5_ZCTAS=2
