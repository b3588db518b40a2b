#!/bin/bash
# round 2 (g): ncu of the c5 block kernel; A/B of the 3-smooth R2C axis in 2-D; host memcpy bandwidth
mkdir -p gpurun_out
python scripts/c5_time.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blocks_tiled -s 3 -c 1 -o gpurun_out/r02g_c5 python scripts/c5_time.py > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
VAR=PCB_MIXED_LAST CFGS="c3 c2" VALS="0 1" bash scripts/ab_env.sh
python - <<'PY'
import numpy as np, time
a = np.random.standard_normal(64 << 20); b = np.empty_like(a)
b[:] = a
t = time.perf_counter()
for _ in range(5): b[:] = a
dt = (time.perf_counter() - t) / 5
print(f"host memcpy (numpy, 1 thread) {a.nbytes / dt / 1e9:.1f} GB/s")
PY
nproc; free -g | head -2
