#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
for c in 2 4; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench$c rc=$?" >> gpurun_out/status.txt; done
for c in 2 3 4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv python bench.py --config $c --batch $([ $c = 4 ] && echo 8 || echo 0) --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_c$c.log 2>&1; echo "ncu-l$c rc=$?" >> gpurun_out/status.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_build -s 3 -c 1 -o gpurun_out/prof_build python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_build.log 2>&1; echo "ncu3 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_c4 python bench.py --config 4 --batch 8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_spmm_c4.log 2>&1; echo "ncu4 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv -s 3 -c 1 -o gpurun_out/prof_spmv_c2 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_spmv_c2.log 2>&1; echo "ncu5 rc=$?" >> gpurun_out/status.txt
