#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp.txt; rm -f $out
python scripts/exp_run.py $out "--config 3|" "--config 3|SPCONV_B200_VARIANT=1" "--config 3|SPCONV_B200_VARIANT=2" "--config 3|SPCONV_B200_VARIANT=3" "--config 3|SPCONV_B200_VARIANT=4" "--config 3|SPCONV_B200_DIAG=1" \
  "--config 4 --batch 8|" "--config 4 --batch 8|SPCONV_B200_VARIANT=1" "--config 4 --batch 8|SPCONV_B200_VARIANT=2" "--config 4 --batch 8|SPCONV_B200_VARIANT=3" "--config 4 --batch 8|SPCONV_B200_VARIANT=4" \
  "--config 4 --batch 64|" "--config 4 --batch 64|SPCONV_B200_VARIANT=2" "--config 4 --batch 64|SPCONV_B200_VARIANT=3" "--config 4 --batch 64|SPCONV_B200_DIAG=1" > /dev/null 2>&1
