#!/bin/bash
# r01e: check kernel (contiguous ranges, unrolled border walk), text I/O tests, densenet bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt gpurun_out/exp.txt
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python scripts/exp_run.py gpurun_out/exp.txt "--config 3|" "--config 3|SPCONV_B200_VARIANT=2" "--config 3|SPCONV_B200_PATH=banded1" \
  "--config 4|" "--config 4|SPCONV_B200_VARIANT=1" "--config 4|SPCONV_B200_PATH=banded1" "--config 4 --batch 64|" \
  "--config 2|" "--config 2|SPCONV_B200_PATH=spmv_plain" > /dev/null 2>&1; echo "exp rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121.md > gpurun_out/bench_densenet.log 2>&1; echo "densenet rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_band_check|conv_spmm_band" -s 6 -c 2 -o gpurun_out/prof_spmm_c3_b256 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu-full-c3 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_band_check|conv_spmm_band" -s 6 -c 2 -o gpurun_out/prof_spmm_c4_b8 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu-full-c4 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv_warp -s 3 -c 1 -o gpurun_out/prof_spmm_c2_b1 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu-full-c2 rc=$?" >> gpurun_out/status.txt
