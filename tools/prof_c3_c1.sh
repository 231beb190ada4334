REPS=1 ncu --set full --clock-control none --import-source on -k regex:"cp_gram|kts_walk" -c 3 -o gpurun_out/prof_c3 -f python tools/cp_c3.py > gpurun_out/ncu_c3full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:glm_run -c 1 -o gpurun_out/prof_c1 -f python tools/glm_probe.py > gpurun_out/ncu_c1full.log 2>&1
tail -1 gpurun_out/ncu_c3full.log; tail -1 gpurun_out/ncu_c1full.log
