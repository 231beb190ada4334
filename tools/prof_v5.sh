#!/bin/bash
# Round-1 v5 profiling pass: bench launch list + ncu --set full captures of the top kernels.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
timeout 600 $CMD > gpurun_out/v5_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v5_launches.csv $CMD > gpurun_out/v5_ncu_launch.log 2>&1
echo "launch list exit $?"
# c2 LMM x16: z-pass (launch 2) and S pass (launch 3) of the second call
REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmm_dmma_kernel -s 2 -c 2 -o gpurun_out/v5_lmm16 -f python tools/lmm16_only.py > gpurun_out/v5_ncu_lmm16.log 2>&1
echo "lmm16 exit $?"
# c2 RMM: colreduce S pass, segsum, R pass
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"colreduce|segsum" -s 3 -c 3 -o gpurun_out/v5_rmm -f python tools/c2_op.py rmm_x1 2 > gpurun_out/v5_ncu_rmm.log 2>&1
echo "rmm exit $?"
# c3 crossprod: fused S pass + walk, R pass, carry fixup
REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cp_gram|cp_carry" -c 3 -o gpurun_out/v5_c3 -f python tools/cp_c3.py > gpurun_out/v5_ncu_c3.log 2>&1
echo "c3 exit $?"
# c1 LogReg cooperative run
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_run -c 1 -o gpurun_out/v5_c1 -f python tools/glm_probe.py > gpurun_out/v5_ncu_c1.log 2>&1
echo "c1 exit $?"
