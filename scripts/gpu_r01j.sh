#!/bin/bash
# r01j: baseline after reverting the PDL apply: variant timings + ncu full of c3 check+apply
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt gpurun_out/exp.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi.txt
timeout 900 python scripts/exp_run.py gpurun_out/exp.txt "--config 3|" "--config 3|SPCONV_B200_VARIANT=2" \
   "--config 4|" "--config 4|SPCONV_B200_VARIANT=1" "--config 3|" > /dev/null 2>&1; echo "exp rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_band_check|conv_spmm_band" -s 6 -c 2 -o gpurun_out/prof_spmm_c3_b256 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu-full-c3 rc=$?" >> gpurun_out/status.txt
