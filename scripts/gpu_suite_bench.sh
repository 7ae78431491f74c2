#!/bin/bash
# GPU parity suite + the default bench line (+ reference arm): gpurun_out/{pytest_gpu,bench,bench_ref}.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python -m pytest -m gpu -q -x ${TESTS:-tests} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
