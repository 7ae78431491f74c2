#!/bin/bash
# ncu --set full of each kernel-choice A/B pair (the variant kept vs the one rejected),
# one launch each, for profiles/r01_choices (scripts/choices_table.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/choices
N="ncu --set full --clock-control none"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 1"
run() { tag=$1; shift; env "$@" > /dev/null; }
# apply blocking (config 3, two-kernel form so the apply is alone): V=16/TH=64 (kept) vs V=8/TH=32 (old)
SPCONV_B200_FUSED=0 timeout 600 $N -k regex:"conv_spmm_band" -s 3 -c 1 -o gpurun_out/choices/apply_v16 $B > /dev/null 2>&1
SPCONV_B200_FUSED=0 SPCONV_B200_VARIANT=11 timeout 600 $N -k regex:"conv_spmm_band" -s 3 -c 1 -o gpurun_out/choices/apply_v8 $B > /dev/null 2>&1
# fused check+apply (kept) vs check kernel (config 3)
timeout 600 $N -k regex:"conv_spmm_band|conv_band_fixup" -s 6 -c 2 -o gpurun_out/choices/fused $B > /dev/null 2>&1
SPCONV_B200_FUSED=0 timeout 600 $N -k regex:"conv_band_check" -s 3 -c 1 -o gpurun_out/choices/check_c3 $B > /dev/null 2>&1
# build write-back: TMA bulk store (kept) vs 16-byte st.global (config 3 block build, config 4 warp build)
timeout 600 $N -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/choices/build3_bulk $B > /dev/null 2>&1
SPCONV_B200_BULK_STORE=0 timeout 600 $N -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/choices/build3_stg $B > /dev/null 2>&1
SPCONV_B200_BUILD=warp timeout 600 $N -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/choices/build4_warp_bulk $B --config 4 > /dev/null 2>&1
SPCONV_B200_BUILD=block timeout 600 $N -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/choices/build4_block_bulk $B --config 4 > /dev/null 2>&1
SPCONV_B200_BUILD=block SPCONV_B200_BULK_STORE=0 timeout 600 $N -k regex:"csr_build" -s 3 -c 1 -o gpurun_out/choices/build4_block_stg $B --config 4 > /dev/null 2>&1
# latency SpMV staging (config 2): per-lane 16-byte loads (kept) vs bulk copies
timeout 600 $N -k regex:"csr_spmv" -s 3 -c 1 -o gpurun_out/choices/spmv_lsu $B --config 2 > /dev/null 2>&1
SPCONV_B200_STAGE=bulk timeout 600 $N -k regex:"csr_spmv" -s 3 -c 1 -o gpurun_out/choices/spmv_bulk $B --config 2 > /dev/null 2>&1
SPCONV_B200_PATH=spmv_plain timeout 600 $N -k regex:"csr_spmv" -s 3 -c 1 -o gpurun_out/choices/spmv_plain $B --config 2 > /dev/null 2>&1
# check kernel for config 4 (one warp per segment, bulk copies)
SPCONV_B200_CHECK=same timeout 600 $N -k regex:"conv_band_check" -s 3 -c 1 -o gpurun_out/choices/check_c4 $B --config 4 > /dev/null 2>&1
ls gpurun_out/choices > gpurun_out/choices/list.txt
# summaries travel back, the reports stay (gpurun_out is capped at 64 MiB)
for r in gpurun_out/choices/*.ncu-rep; do python scripts/ncu_summary.py "$r" --json "${r%.ncu-rep}.json" > "${r%.ncu-rep}.txt" 2>&1; done
rm -f gpurun_out/choices/*.ncu-rep
