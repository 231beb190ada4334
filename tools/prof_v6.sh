#!/bin/bash
# Round-1 v6 profiling pass (after the two-barrier GD run and the narrow gram): bench launch list,
# ncu --set full of the c1 GD run and of the c5 GNMF step kernels.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
timeout 600 $CMD > gpurun_out/v6_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v6_launches.csv $CMD > gpurun_out/v6_ncu_launch.log 2>&1
echo "launch list exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_run -c 1 -o gpurun_out/v6_c1 -f python tools/glm_probe.py > gpurun_out/v6_ncu_c1.log 2>&1
echo "c1 exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"narrow_gram|lmm_dmma|nmf_update|segsum|colreduce" -s 8 -c 6 -o gpurun_out/v6_c5 -f python tools/workload.py c5 1 > gpurun_out/v6_ncu_c5.log 2>&1
echo "c5 exit $?"
