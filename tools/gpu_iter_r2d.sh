#!/bin/bash
TAG=${1:-r2d}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -ra > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python tools/small_jobs.py > gpurun_out/small_jobs_$TAG.jsonl 2> gpurun_out/small_jobs_$TAG.err
QK_SHORT_CHAIN=0 timeout 600 python tools/small_jobs.py > gpurun_out/small_jobs_${TAG}_noshort.jsonl 2>&1
for v in 0 3 4; do
  QK_GATE_VARIANT=$v timeout 300 ncu --set full --clock-control none -k regex:gate_build -c 1 \
    -o gpurun_out/prof_gate_${TAG}_v$v python tools/gate_bench.py > gpurun_out/ncu_gate_${TAG}_v$v.log 2>&1
done
QK_TRACE=1 timeout 300 python tools/e2e_trace.py 5 --pageable > gpurun_out/trace_pageable_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 \
  -o gpurun_out/prof_sweep16_$TAG python tools/small_jobs.py --only c5_16 --reps 1 > gpurun_out/ncu_sweep16_$TAG.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo done
