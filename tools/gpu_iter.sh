#!/bin/bash
# Iteration call: gpu tests, bench (variants via QK_SWEEP_RI), ncu capture of one Gram sweep.
TAG=${1:-it}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for RI in 4 2; do
  QK_SWEEP_RI=$RI timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_ri$RI.json 2> gpurun_out/bench_${TAG}_ri$RI.err
done
for RI in ${NCU_RI:-4}; do
  QK_SWEEP_RI=$RI timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 \
    -o gpurun_out/prof_sweep_${TAG}_ri$RI python tools/profile_sweep.py > gpurun_out/ncu_${TAG}_ri$RI.log 2>&1
done
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe_$TAG.json 2>&1
echo done
