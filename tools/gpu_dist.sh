#!/bin/bash
# distributed-pass checks on one GPU: emulated parts bitwise, the 2-rank bench smoke, per-rank estimate
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_scale.py tests/test_gpu_bench_smoke.py > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dist.log
timeout 900 python tools/dist_estimate.py 2 4 8 > gpurun_out/dist_estimate.log 2>&1; echo "estimate rc=$?"; grep -v "^{" gpurun_out/dist_estimate.log | tail -6
