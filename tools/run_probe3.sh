cd $GRAFT_REPO_ROOT
for nr in 100000 1000000; do for d in 0 1 2 3 4; do echo "NR=$nr debug=$d"; NR=$nr FB_LMM_DEBUG=$d timeout 120 python tools/time_lmm.py 2>&1 | tail -1; done; done
