#!/bin/bash
# One gpurun call: GPU tests + smoke, then the every-entry parity report over configs 1-4.
# usage: gpurun --timeout 5400 -- 'bash tools/gpu_parity_r2.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nproc > gpurun_out/host_r2p.txt; lscpu >> gpurun_out/host_r2p.txt; free -g >> gpurun_out/host_r2p.txt
timeout 1500 python -m pytest tests -m gpu -q -ra -x > gpurun_out/pytest_gpu_r2p.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_r2p.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2p.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_r2p.log
timeout 4800 python tools/parity_report.py gpurun_out/r2_parity.json > gpurun_out/parity_r2.log 2>&1
echo "parity exit $?" >> gpurun_out/parity_r2.log
echo done
