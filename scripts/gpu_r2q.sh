#!/bin/bash
mkdir -p gpurun_out
CFGS="c3 c2 c4" bash scripts/ab_bench.sh
CFGS="c3" bash scripts/ab_bench.sh
