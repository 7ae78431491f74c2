#!/usr/bin/env python
"""Tuning-experiment driver: runs bench.py under several env settings and prints
one summary line each.   python scripts/exp_run.py OUT 'ARGS|ENV=V ENV2=V' ..."""
import json
import os
import subprocess
import sys

out = sys.argv[1]
with open(out, "a") as f:
    for spec in sys.argv[2:]:
        args, _, envs = spec.partition("|")
        env = dict(os.environ)
        for kv in envs.split():
            k, _, v = kv.partition("=")
            env[k] = v
        cmd = [sys.executable, "bench.py", "--steps", "40", "--warmup", "3", "--no-cpu-baseline",
               "--e2e-steps", "2", "--no-secondary"] + args.split()
        try:
            r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
            j = json.loads(r.stdout.strip().splitlines()[-1])
            line = (f"{spec:60s} {j['ms_per_step'] * 1e3:9.1f} us  frac {j['roofline']['frac']:.3f}  "
                    f"build {j['build']['ms_device'] * 1e3:.1f} us  e2e {j['e2e']['value']:.1f}  "
                    f"{j['roofline']['kernel']}")
        except Exception as e:  # noqa: BLE001
            line = f"{spec:60s} FAILED {type(e).__name__}: {(r.stderr if 'r' in dir() else '')[-300:]}"
        print(line)
        f.write(line + "\n")
        f.flush()
