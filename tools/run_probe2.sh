cd $GRAFT_REPO_ROOT
for b in 200 100 72; do for mt in 0 2 1; do echo "budget=$b mt=$mt"; FB_RING_BUDGET_KB=$b FB_LMM_MT=$mt timeout 120 python tools/time_lmm.py; done; done
echo "NR=500k"; NR=500000 timeout 120 python tools/time_lmm.py
echo "NR=250k"; NR=250000 timeout 120 python tools/time_lmm.py
echo "NR=100k"; NR=100000 timeout 120 python tools/time_lmm.py
