cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python scripts/probe_f64.py > gpurun_out/probe_f64.log 2>&1; echo "probe rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 30 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_spmm_band|conv_band_check" -c 4 -o gpurun_out/prof_csc_c3 python scripts/csc_ncu.py > gpurun_out/ncu_csc.log 2>&1; echo "ncu rc=$?" >> gpurun_out/status.txt
