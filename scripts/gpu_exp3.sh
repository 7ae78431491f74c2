#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp.txt; rm -f $out
run() { echo "== $BARGS $*" >> $out; env "$@" timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 2 $BARGS 2>&1 | tail -1 | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step']*1000,1),'us', round(j['roofline']['frac'],3))" >> $out 2>&1; }
BARGS="--config 3"; for v in 0 1 2 3 4; do run SPCONV_B200_VARIANT=$v; done; run SPCONV_B200_VARIANT=1 SPCONV_B200_SPLITS=1
BARGS="--config 4 --batch 8"; for v in 0 1 2 3 4; do run SPCONV_B200_VARIANT=$v; done
BARGS="--config 4 --batch 64"; for v in 0 1 3; do run SPCONV_B200_VARIANT=$v; done
