cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest -m gpu -q -x ${TESTS:-tests} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python scripts/ab_fused.py > gpurun_out/ab_fused.log 2>&1; echo "ab rc=$?" >> gpurun_out/status.txt
