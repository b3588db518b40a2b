#!/bin/bash
# round 2 (b): new tests, c5 timing, c3/c4 launch lists with DRAM bytes, ncu --set full of cols
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long_lines.py tests/test_gpu_headline.py tests/test_gpu_tools.py -q -p no:cacheprovider -k "not fft_engine" > gpurun_out/pytest_b.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_b.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; tail -3 gpurun_out/c5.log
for cfg in c3 c4; do
  CMD="python bench.py --config $cfg --profile-only --steps 2 --warmup 3"
  $CMD > gpurun_out/plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_r02b_$cfg.csv $CMD > gpurun_out/ncu_launch_$cfg.log 2>&1
  echo "launch list $cfg rc=$?"
done
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cols -s 3 -c 1 -o gpurun_out/r02b_c3_cols $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
