#!/bin/bash
# Final round-2 evidence on the frozen build: launch lists with DRAM bytes (-> traffic json with the
# build's source hash), ncu --set full of the top cols and gather launches, bench lines, reference arm.
mkdir -p gpurun_out/final
for cfg in c3 c4; do
  CMD="python bench.py --config $cfg --profile-only --steps 2 --warmup 3"
  $CMD > gpurun_out/final/plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/final/launches_$cfg.csv $CMD > gpurun_out/final/ncu_launch_$cfg.log 2>&1
  echo "launch list $cfg rc=$?"
done
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_cols<256, 4, 1>" -s 2 -c 1 -o gpurun_out/final/c3_cols256 $CMD > gpurun_out/final/ncu_cols.log 2>&1
echo "ncu cols rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_rows_inv_b<128" -s 2 -c 1 -o gpurun_out/final/c3_rows_inv_b $CMD > gpurun_out/final/ncu_rinv.log 2>&1
echo "ncu rows_inv rc=$?"
for cfg in c1 c2 c4 c3; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/final/bench_$cfg.json 2> gpurun_out/final/bench_$cfg.err
  echo "bench $cfg rc=$?"
done
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/ref_c3.json 2> gpurun_out/final/ref_c3.err
echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 300 python scripts/c5_time.py > gpurun_out/final/c5.log 2>&1; cp gpurun_out/c5_time.json gpurun_out/final/ 2>/dev/null
timeout 600 python scripts/estimator_time.py > gpurun_out/final/est.log 2>&1; cp gpurun_out/estimator_c3.json gpurun_out/final/ 2>/dev/null
echo done
