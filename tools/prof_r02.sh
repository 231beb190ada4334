#!/bin/bash
# Round-2 pass: GPU tests, smoke, default bench, the reference arm, the bench launch list and
# ncu --set full captures (summarised on the box; reports stay in /tmp there) of the c2 LMM x16 /
# RMM kernels, the c3 crossprod kernels and the c4/c5 driver steps.
# usage: tools/prof_r02.sh TAG [tests=1] [ncu=1]
set -u
T=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
if [ "${2:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?"
  tail -3 gpurun_out/${T}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke exit $?"
fi
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref exit $?"
full() {  # name, "ncu filter args", command...
  local name=$1 filt=$2; shift 2
  timeout 900 ncu --set full --clock-control none $filt -o /tmp/${T}_${name} -f "$@" > gpurun_out/${T}_ncu_${name}.log 2>&1
  echo "$name exit $?"
  python tools/ncu_summary.py /tmp/${T}_${name}.ncu-rep "${T} ${name}" > gpurun_out/${T}_ncu_${name}.txt 2>&1
}
if [ "${3:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
  echo "launch list exit $?"
  full lmm16 "-k regex:lmm_ -s 2 -c 2" python tools/c2_op.py lmm_x16 2
  full rmm "-k regex:colreduce|lmm_|rows_wt|segsum|rth -s 2 -c 4" python tools/c2_op.py rmm_x1 3
  REPS=2 full c3 "-k regex:cp_ -s 4 -c 4" python tools/cp_c3.py
  full c4 "-k regex:kmeans_|rth_ -s 6 -c 6" python tools/time_kmeans.py
  full c5 "-k regex:nmf_|rth_|narrow_gram -s 10 -c 10" python tools/time_gnmf.py
fi
