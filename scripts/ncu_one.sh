#!/bin/bash
# ncu --set full on the first launch matching each demangled-name regex: ncu_one.sh "re1;re2" <bench args>
RES=$1; shift
CMD="python bench.py --profile-only --steps 1 --warmup 1 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain.log; exit 1; }
i=0
IFS=';' read -ra ARR <<< "$RES"
for re in "${ARR[@]}"; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -c 1 \
      -o gpurun_out/one_$i $CMD > gpurun_out/ncu_$i.log 2>&1
  echo "ncu[$i] rc=$? $re"; i=$((i+1))
done
