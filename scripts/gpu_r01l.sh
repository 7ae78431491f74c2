#!/bin/bash
# r01l: latency SpMV staging A/B (bulk vs lsu), c2 warm/cold, densenet both, CSC secondary
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt gpurun_out/exp.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python scripts/exp_run.py gpurun_out/exp.txt "--config 2|" "--config 2|SPCONV_B200_STAGE=lsu" "--config 2|SPCONV_B200_PATH=spmv_plain" > /dev/null 2>&1; echo "exp rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_sec.log 2>&1; echo "bench-sec rc=$?" >> gpurun_out/status.txt
SPCONV_B200_STAGE=lsu timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_sec_lsu.log 2>&1; echo "bench-sec-lsu rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121.md > gpurun_out/bench_densenet.log 2>&1; echo "densenet rc=$?" >> gpurun_out/status.txt
SPCONV_B200_STAGE=lsu timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121_lsu.md > gpurun_out/bench_densenet_lsu.log 2>&1; echo "densenet-lsu rc=$?" >> gpurun_out/status.txt
