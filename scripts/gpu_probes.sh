#!/bin/bash
# The round's A/B probes (kernel-choice evidence): fused vs two-kernel band
# forms, latency SpMV kernels, off-band geometries, fp64 apply, host-path
# anatomy, build kernels, batch scaling, CSC checks, odd widths, grouped
# calls, write bandwidth -> gpurun_out/probes/
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/probes
timeout 600 python scripts/ab_fused.py 20 > gpurun_out/probes/ab_fused.txt 2>&1
timeout 600 python scripts/probe_spmv.py > gpurun_out/probes/probe_spmv.txt 2>&1
timeout 600 python scripts/probe_geoms.py 10 > gpurun_out/probes/probe_geoms.txt 2>&1
timeout 600 python scripts/probe_f64.py > gpurun_out/probes/probe_f64.txt 2>&1
timeout 300 python scripts/probe_host.py > gpurun_out/probes/probe_host.txt 2>&1
timeout 600 python scripts/build_ab.py 30 > gpurun_out/probes/build_ab.txt 2>&1
timeout 600 python scripts/probe_batch_scaling.py > gpurun_out/probes/probe_batch_scaling.txt 2>&1
timeout 600 python scripts/probe_csc_check.py > gpurun_out/probes/probe_csc_check.txt 2>&1
timeout 600 python scripts/probe_notma.py > gpurun_out/probes/probe_notma.txt 2>&1
timeout 300 python scripts/probe_group.py > gpurun_out/probes/probe_group.txt 2>&1
timeout 300 python scripts/probe_write_peak.py > gpurun_out/probes/probe_write_peak.txt 2>&1
echo done > gpurun_out/probes/status.txt
