#!/bin/bash
# round 2 sweep on the final build: apply vs adjoint (c3, c4), the GLOBAL plan (c3, c4), k-shard
# path at world size 1 through torchrun (the library's NCCL reduce on a 1-rank communicator)
mkdir -p gpurun_out/sweep
python scripts/adjoint_time.py c3 64 > gpurun_out/sweep/adjoint_c3.json 2>&1; tail -1 gpurun_out/sweep/adjoint_c3.json
python scripts/adjoint_time.py c4 8 > gpurun_out/sweep/adjoint_c4.json 2>&1; tail -1 gpurun_out/sweep/adjoint_c4.json
for cfg in c3 c4; do
  timeout 900 python bench.py --config $cfg --mode global --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/global_$cfg.json 2> gpurun_out/sweep/global_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/sweep/global_$cfg.json'));print('$cfg global', round(d['value'],1), round(d['roofline']['frac'],3), d['kernels_ms_per_step'])"
done
PCB_BENCH_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/dist1_c3.json 2> gpurun_out/sweep/dist1_c3.err
python -c "import json;d=json.load(open('gpurun_out/sweep/dist1_c3.json'));print('dist1 c3', round(d['value']), d['plan']['reduce'], d['e2e']['value'])" || tail -5 gpurun_out/sweep/dist1_c3.err
