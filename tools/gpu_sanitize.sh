#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_smoke.py, then the
# randomised host-pipeline stress.  usage: gpurun --timeout 2400 -- 'bash tools/gpu_sanitize.sh TAG'
TAG=${1:-r2}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py \
    > gpurun_out/sanitizer/${TAG}_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer/${TAG}_$tool.log
done
timeout 700 python tools/stress_pipelines.py 600 > gpurun_out/stress_$TAG.log 2>&1
echo "stress exit $?" >> gpurun_out/stress_$TAG.log
echo done
