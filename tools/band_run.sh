#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -q -m gpu -k "band_layout" > gpurun_out/band_pytest.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/band_pytest.log
{
for dbg in 0 8; do echo "== FB_LMM_DEBUG=$dbg"; FB_LMM_DEBUG=$dbg timeout 300 python tools/lmm_band_exp.py; done
echo "== DX=8"; DX=8 timeout 300 python tools/lmm_band_exp.py
} > gpurun_out/band_exp3.log 2>&1
cat gpurun_out/band_exp3.log
