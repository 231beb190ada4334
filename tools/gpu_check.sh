#!/bin/bash
# One gpurun pass: GPU tests, smoke, bench, launch list, ncu full capture of the top kernels.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
if [ "${4:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
  timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  echo "launch list exit $?" >> gpurun_out/ncu_launch.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${1:-lmm_|colreduce}" -s ${2:-2} -c ${3:-4} -o gpurun_out/prof -f $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/ncu_full.log
fi
