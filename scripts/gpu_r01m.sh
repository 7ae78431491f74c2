#!/bin/bash
# r01m: full bench line, ncu of c2 latency SpMV (lsu) and of the CSC build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv -s 3 -c 1 -o gpurun_out/prof_spmm_c2_b1 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 2 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu-full-c2 rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csc_build -c 1 -o gpurun_out/prof_cscbuild_c3 python -c "
import numpy as np, torch, paper_2411_19419_b200 as sp
t = sp.build_transform(sp.Kernel(3, np.ones(9)), sp.ConvSpec(1024, 1024, 3, 1, 1), layout=sp.Layout.CSC)
torch.cuda.synchronize()" > gpurun_out/ncu_cscbuild.log 2>&1; echo "ncu-cscbuild rc=$?" >> gpurun_out/status.txt
