#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp.txt; rm -f $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "banded or spmm or spmv" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out
run() { echo "== $BARGS $*" >> $out; env "$@" timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 2 $BARGS 2>&1 | tail -1 | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step']*1000,1),'us', round(j['roofline']['frac'],3))" >> $out 2>&1; }
BARGS="--config 3"; run X=0; run SPCONV_B200_DIAG=1; run SPCONV_B200_SPLITS=1
BARGS="--config 4 --batch 8"; run X=0; run SPCONV_B200_DIAG=1
BARGS="--config 4 --batch 64"; run X=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_c4 python bench.py --config 4 --batch 8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_spmm_c4.log 2>&1; echo "ncu4 rc=$?" >> $out
