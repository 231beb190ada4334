cd $GRAFT_REPO_ROOT
for lib in "" build/cg/libfactorla_b200.so; do for mt in 2 4; do for nr in 1000000 100000; do echo "lib=$lib mt=$mt NR=$nr"; FB_LIB_PATH=$lib FB_LMM_MT=$mt NR=$nr timeout 120 python tools/time_lmm.py 2>&1 | tail -1; done; done; done
