set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ml_gpu.py -q -m gpu -x -k "kmeans" 2>&1 | tail -2
for v in "" "FB_KM_ONEHOT_LANES=1"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:onehot --log-file gpurun_out/oh.csv python tools/workload.py c4 1 > /dev/null 2>&1
  echo "[$v]"; python tools/launches.py gpurun_out/oh.csv | head -3
done
