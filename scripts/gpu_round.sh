#!/bin/bash
# Round evidence: parity suite, smoke, bench (our arm + reference arm), DenseNet table,
# launch list of the default bench, ncu --set full of every hot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi -L > gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench-ref rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121.md > gpurun_out/bench_densenet.log 2>&1; echo "densenet rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_launch_c3.log 2>&1; echo "ncu-l3 rc=$?" >> gpurun_out/status.txt
# config 3 runs the fused check+apply + fixup per call: skip the 3 warm-up calls, capture one timed call
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_spmm_band|conv_band_fixup" -s 6 -c 2 -o gpurun_out/prof_spmm_c3_b256 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu-full-c3 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_band_check|conv_spmm_band" -s 6 -c 2 -o gpurun_out/prof_spmm_c4_b8 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu-full-c4 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv -s 3 -c 1 -o gpurun_out/prof_spmm_c2_b1 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu-full-c2 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/prof_build_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_build3.log 2>&1; echo "ncu-full-build3 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/prof_build_c4 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_build4.log 2>&1; echo "ncu-full-build4 rc=$?" >> gpurun_out/status.txt
timeout 900 python scripts/exp_run.py gpurun_out/exp.txt "--config 3|" "--config 3 --batch 1024|" "--config 4|" "--config 4 --batch 64|" "--config 2|" "--config 3|SPCONV_B200_FUSED=0" > /dev/null 2>&1; echo "exp rc=$?" >> gpurun_out/status.txt
# multi-rank path on the one GPU (2 ranks sharing it over gloo): barrier, max-over-ranks, gather
SPCONV_B200_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 --gather > gpurun_out/bench_2rank_gloo.log 2>&1; echo "2rank rc=$?" >> gpurun_out/status.txt
timeout 300 python scripts/zt_probe.py > gpurun_out/zt.txt 2>&1; echo "zt rc=$?" >> gpurun_out/status.txt
