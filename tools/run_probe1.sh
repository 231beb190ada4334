cd $GRAFT_REPO_ROOT
tools/red_probe > gpurun_out/red.log 2>&1
for sf in 1.0 0.5; do for gf in 0 1.0 0.5 0.7; do FB_ZSTORE_FRAC=$sf FB_ZGATHER_FRAC=$gf timeout 120 python tools/time_lmm.py; done; done > gpurun_out/lmm.log 2>&1
FB_ZSTORE_FRAC=1.0 FB_ZGATHER_FRAC=0.6 timeout 120 python tools/time_lmm.py >> gpurun_out/lmm.log 2>&1
FB_ZSTORE_FRAC=0.6 FB_ZGATHER_FRAC=0.6 timeout 120 python tools/time_lmm.py >> gpurun_out/lmm.log 2>&1
cat gpurun_out/red.log gpurun_out/lmm.log
