cd $GRAFT_REPO_ROOT
for nr in 100000; do for cfg in "200 4" "224 4"; do set -- $cfg; echo "NR=$nr budget=$1 mt=$2"; NR=$nr FB_RING_BUDGET_KB=$1 FB_LMM_MT=$2 timeout 120 python tools/time_lmm.py 2>&1 | tail -1; NR=$nr FB_LMM_DEBUG=3 FB_RING_BUDGET_KB=$1 FB_LMM_MT=$2 timeout 120 python tools/time_lmm.py 2>&1 | tail -1; done; done
