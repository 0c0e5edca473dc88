#!/bin/bash
# gate-build microbench, small-job probe, pageable e2e trace, parity configs 1-2 re-run
TAG=${1:-r2b}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -ra > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python tools/gate_bench.py > gpurun_out/gate_bench_$TAG.jsonl 2>&1
timeout 600 python tools/small_jobs.py > gpurun_out/small_jobs_$TAG.jsonl 2> gpurun_out/small_jobs_$TAG.err
QK_TRACE=1 timeout 300 python tools/e2e_trace.py 4 --pageable > gpurun_out/trace_pageable_$TAG.log 2>&1
QK_TRACE=1 timeout 300 python tools/e2e_trace.py 4 > gpurun_out/trace_pinned_$TAG.log 2>&1
cp profiles/r2_parity.json gpurun_out/r2_parity_in.json
timeout 600 python tools/parity_report.py gpurun_out/r2_parity_c12.json --configs 1,2 --merge gpurun_out/r2_parity_in.json > gpurun_out/parity_c12_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate_build -c 2 \
  -o gpurun_out/prof_gate_$TAG python tools/gate_bench.py > gpurun_out/ncu_gate_$TAG.log 2>&1
echo done
