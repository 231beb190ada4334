for dbg in 0 1 2 3; do
FB_CP_DEBUG=$dbg REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"cp_gram|kts_walk" --log-file gpurun_out/ll_$dbg.csv python tools/cp_c3.py > /dev/null 2>&1
done
