#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_ml_gpu.py -q -m gpu -x -k "band or kmeans" > gpurun_out/band_pytest.log 2>&1; echo "pytest exit $?"
tail -4 gpurun_out/band_pytest.log
timeout 600 python tools/km_band_ab.py > gpurun_out/km_band_ab.log 2>&1
cat gpurun_out/km_band_ab.log
