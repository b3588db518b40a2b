#!/bin/bash
# env-var sweep of the local pipeline knobs on c3
for env in "PCB_PIPELINE=0" "PCB_PIPELINE=1" "PCB_PIPELINE=0 PCB_CHUNK_TERMS=1000" "PCB_PIPELINE=1 PCB_CHUNK_TERMS=16" "PCB_PIPELINE=1 PCB_CHUNK_TERMS=8"; do
  echo "== $env"
  env $env bash scripts/gpu_check.sh "$@" 2>&1 | tail -1
done
