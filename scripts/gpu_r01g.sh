#!/bin/bash
# r01g: CSC + device verify sweep parity, densenet per-layer table
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121.md > gpurun_out/bench_densenet.log 2>&1; echo "densenet rc=$?" >> gpurun_out/status.txt
