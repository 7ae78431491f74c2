#!/bin/bash
# Round evidence (round 2): parity suite, smoke, bench (our arm + reference arm),
# DenseNet table, the 2-rank path, the launch list of the default bench, and an
# ncu --set full capture of every hot kernel (scripts/ncu_target.py).
# Then: python scripts/make_profiles.py <tag>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi -L > gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench-ref rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --workload densenet121 --steps 100 --warmup 10 --report gpurun_out/densenet121.md > gpurun_out/bench_densenet.log 2>&1; echo "densenet rc=$?" >> gpurun_out/status.txt
SPCONV_B200_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 --gather > gpurun_out/bench_2rank_gloo.log 2>&1; echo "2rank rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_launch_c3.log 2>&1; echo "ncu-launches rc=$?" >> gpurun_out/status.txt
nc() {  # name regex skip count target
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c $4 -o gpurun_out/$1 python scripts/ncu_target.py $5 3 > gpurun_out/ncu_$1.log 2>&1; echo "ncu $1 rc=$?" >> gpurun_out/status.txt
}
nc prof_spmm_c3_b256 "conv_spmm_band" 3 1 c3
nc prof_spmm_c3_b32 "conv_spmm_band" 3 1 c3b32
nc prof_csc_c3_b256 "conv_spmm_band" 3 1 c3csc
nc prof_f64_c3_b256 "conv_band_check|conv_spmm_band" 6 2 c3f64
nc prof_spmm_c4_b8 "conv_band_check|conv_spmm_band" 6 2 c4
nc prof_spmm_c2_b1 "conv_spmv_win" 3 1 c2
nc prof_build_c3 "csr_build" 3 1 build3
nc prof_build_c4 "csr_build" 3 1 build4
nc prof_k11_c5_b256 "conv_band_check|conv_spmm_band" 6 2 c5k11
nc prof_group_densenet "csr_spmv_group" 3 1 group
# the reports are large: summarise them on the box and bring back the text
TAG=${TAG:-r02}
python scripts/make_profiles.py $TAG gpurun_out > gpurun_out/make_profiles.log 2>&1
mkdir -p gpurun_out/profiles_out && cp -r profiles/$TAG gpurun_out/profiles_out/
for f in gpurun_out/*.ncu-rep; do [ -f "$f" ] && [ $(stat -c %s "$f") -gt 8000000 ] && rm -f "$f"; done
echo "done" >> gpurun_out/status.txt
