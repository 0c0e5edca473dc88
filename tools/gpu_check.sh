#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the sweep kernel.
# usage (from the build container): gpurun --timeout 1800 -- 'bash tools/gpu_check.sh [tag]'
TAG=${1:-r1}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/clocks_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 \
  -o gpurun_out/prof_sweep_$TAG python bench.py --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate_build -c 1 \
  -o gpurun_out/prof_gate_$TAG python bench.py --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/ncu_gate_$TAG.log 2>&1
fi
echo done
