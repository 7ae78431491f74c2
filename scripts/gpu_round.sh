#!/bin/bash
# One GPU session: gpu parity tests, benches (c3 default + c2 + c4), reference arm,
# ncu launch lists and --set full captures of the top kernels.  Results -> gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench_ref rc=$?" >> gpurun_out/status.txt
for c in 2 4; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench$c rc=$?" >> gpurun_out/status.txt; done
for c in 2 3 4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv python bench.py --config $c --batch $([ $c = 4 ] && echo 8 || echo 0) --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_c$c.log 2>&1; echo "ncu-l$c rc=$?" >> gpurun_out/status.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu-full-c3 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_build -s 3 -c 1 -o gpurun_out/prof_build_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_build.log 2>&1; echo "ncu-full-build rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_c4 python bench.py --config 4 --batch 8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu-full-c4 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv -s 3 -c 1 -o gpurun_out/prof_spmv_c2 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu-full-c2 rc=$?" >> gpurun_out/status.txt
