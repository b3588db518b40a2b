#!/bin/bash
# Round-2 final evidence on the frozen build (session 3): GPU test suite, launch lists with DRAM bytes
# (-> traffic json with the build's source hash), ncu --set full of the top cols and gather launches
# (summaries exported here; the reports are too large to bring back), bench lines of every config,
# the reference arm, c5 / estimator / H-matrix timings, headline parity numbers, smoke.
O=gpurun_out/final; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/gputest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/gputest.log)"
for cfg in c3 c4; do
  CMD="python bench.py --config $cfg --profile-only --steps 2 --warmup 3"
  $CMD > $O/plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_$cfg.csv $CMD > $O/ncu_launch_$cfg.log 2>&1
  echo "launch list $cfg rc=$?"
  python scripts/launch_share.py $O/launches_$cfg.csv 5 > $O/${cfg}_launches_share.txt
done
python scripts/traffic_json.py $O/launches_c3.csv 5 $O/traffic_c3_local.json 64
python scripts/traffic_json.py $O/launches_c4.csv 5 $O/traffic_c4_local.json 8
cp $O/traffic_c3_local.json $O/traffic_c4_local.json profiles/   # bench reads profiles/traffic_*.json
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3"
cap() { # tag regex
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s 2 -c 1 \
      -f -o /tmp/ncu_$1 $CMD > $O/ncu_$1.log 2>&1
  echo "ncu $1 rc=$?"
  { python scripts/ncu_summary.py /tmp/ncu_$1.ncu-rep; python scripts/ncu_hot.py /tmp/ncu_$1.ncu-rep 20; } > $O/c3_top_$1_full.txt 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page details > $O/c3_top_$1_details.txt 2>/dev/null
}
cap cols 'k_cols<\(int\)256, \(int\)4, \(int\)1>'
cap rows_inv_b 'k_rows_inv_b<\(int\)128, \(int\)4, \(int\)0>'
for cfg in c1 c2 c4 c3; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  echo "bench $cfg rc=$?"
done
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_c3.json 2> $O/ref_c3.err
echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"
for a in adjoint global; do :; done
timeout 300 python scripts/c5_time.py > $O/c5.log 2>&1; cp gpurun_out/c5_time.json $O/ 2>/dev/null
PCB_BLOCKS_STREAMS=1 timeout 300 python scripts/c5_time.py > $O/c5_one_stream.log 2>&1; cp gpurun_out/c5_time.json $O/c5_time_one_stream.json 2>/dev/null
timeout 600 python scripts/estimator_time.py > $O/est.log 2>&1; cp gpurun_out/estimator_c3.json $O/ 2>/dev/null
timeout 900 python scripts/hmatrix_time.py > $O/hmatrix.log 2>&1; cp gpurun_out/hmatrix_time.json $O/ 2>/dev/null
timeout 900 python scripts/adjoint_time.py > $O/adjoint.log 2>&1; cp gpurun_out/adjoint*.json $O/ 2>/dev/null
python scripts/headline_errors.py > $O/hp.log 2>&1; cp gpurun_out/headline_parity.json $O/ 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
du -sh gpurun_out
echo done
