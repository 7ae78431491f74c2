#!/bin/bash
# tuning experiments (diagnostic knobs; never used by the product defaults)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp.txt; rm -f $out
run() { echo "== $*" >> $out; env "$@" timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 2 $BARGS 2>&1 | tail -1 | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step']*1000,1),'us', round(j['roofline']['frac'],3))" >> $out 2>&1; }
BARGS="--config 3"
run X=0
run SPCONV_B200_DIAG=1
for sp in 1 2 4 8 16; do run SPCONV_B200_SPLITS=$sp; done
BARGS="--config 4 --batch 8"
run X=0
run SPCONV_B200_DIAG=1
run SPCONV_B200_PATH=tiled
BARGS="--config 4 --batch 64"
run X=0
run SPCONV_B200_DIAG=1
