#!/bin/bash
# r01r: speculative-gather latency SpMV -- parity, config 2 cold/warm A/B, DenseNet table, ncu
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt gpurun_out/exp.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python scripts/exp_run.py gpurun_out/exp.txt "--config 2|" "--config 2|SPCONV_B200_SPMV=bulk" > /dev/null 2>&1; echo "exp rc=$?" >> gpurun_out/status.txt
for v in spec bulk; do SPCONV_B200_SPMV=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_sec_$v.log 2>&1; echo "bench-$v rc=$?" >> gpurun_out/status.txt; done
timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121.md > gpurun_out/bench_densenet.log 2>&1; echo "densenet rc=$?" >> gpurun_out/status.txt
SPCONV_B200_SPMV=bulk timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121_bulk.md > gpurun_out/bench_densenet_bulk.log 2>&1; echo "densenet-bulk rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv -s 3 -c 1 -o gpurun_out/prof_spmm_c2_b1 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu-full-c2 rc=$?" >> gpurun_out/status.txt
