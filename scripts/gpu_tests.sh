#!/bin/bash
# GPU parity suite (optionally a subset: pytest arguments) -> gpurun_out/pytest_gpu.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout ${T:-1200} python -m pytest -m gpu -q -x --durations=10 "${@:-tests}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/status.txt
