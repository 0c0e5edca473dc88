#!/bin/bash
# Round-2 iteration call: GPU tests, smoke, small-job probe, short bench, ncu of the gate build
# and a launch list of the C2 job.   usage: gpurun -- 'bash tools/gpu_iter_r2.sh TAG'
TAG=${1:-it}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -ra > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 600 python tools/small_jobs.py > gpurun_out/small_jobs_$TAG.jsonl 2> gpurun_out/small_jobs_$TAG.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2_$TAG.csv python tools/small_jobs.py --only c2 --reps 2 \
  > gpurun_out/ncu_c2_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gate_build -c 1 \
  -o gpurun_out/prof_gate_$TAG python bench.py --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/ncu_gate_$TAG.log 2>&1
echo done
