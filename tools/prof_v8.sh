#!/bin/bash
# Round-1 final pass: GPU tests, smoke, default bench, the reference arm, the bench launch list and
# one ncu --set full capture of the c3 crossprod kernels (fused S pass + R pass).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/v8_pytest.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/v8_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v8_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/v8_bench.json 2> gpurun_out/v8_bench.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/v8_bench_ref.json 2> gpurun_out/v8_bench_ref.err; echo "ref exit $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v8_launches.csv $CMD > gpurun_out/v8_ncu_launch.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_gram -c 2 -o gpurun_out/v8_c3 -f python tools/cp_c3.py > gpurun_out/v8_ncu_c3.log 2>&1
echo "c3 exit $?"
