#!/bin/bash
# quick iteration: gpu parity tests + A/B timings (+ optional ncu of one kernel: NCU_K regex, NCU_ARGS bench args)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt gpurun_out/exp.txt
timeout 600 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python scripts/exp_run.py gpurun_out/exp.txt "$@" > /dev/null 2>&1; echo "exp rc=$?" >> gpurun_out/status.txt
if [ -n "$NCU_K" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s 4 -c 2 -o gpurun_out/prof_quick python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 1 $NCU_ARGS > gpurun_out/ncu_quick.log 2>&1; echo "ncu rc=$?" >> gpurun_out/status.txt
fi
