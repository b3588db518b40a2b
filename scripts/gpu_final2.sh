#!/bin/bash
bash scripts/gpu_final.sh
bash scripts/gpu_final_ncu.sh
python scripts/headline_errors.py > gpurun_out/final/hp.log 2>&1; cp gpurun_out/headline_parity.json gpurun_out/final/ 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
