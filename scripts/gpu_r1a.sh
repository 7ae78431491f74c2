#!/bin/bash
# first GPU pass: smoke, gpu tests, bench, ncu launch list + full captures
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench2 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_spmm -s 3 -c 1 -o gpurun_out/prof_spmm python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_spmm.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_build -s 3 -c 1 -o gpurun_out/prof_build python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_build.log 2>&1; echo "ncu3 rc=$?" >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/pytest_slow.log 2>&1; echo "slow rc=$?" >> gpurun_out/status.txt
