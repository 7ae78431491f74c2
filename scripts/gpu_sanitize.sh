#!/bin/bash
# compute-sanitizer over the round-2 kernels (memcheck; racecheck / synccheck on
# the band tests): gpurun_out/sanitize/
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/sanitize
T="tests/test_gpu_csc_native.py tests/test_gpu_f64_band.py tests/test_gpu_band_geoms.py tests/test_gpu_group.py"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -m gpu -q -x $T -k "not full_size" > gpurun_out/sanitize/memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize/status.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -m gpu -q -x tests/test_gpu_csc_native.py tests/test_gpu_group.py -k "band_forms or detects_interior or group_matches or f64_bitexact" > gpurun_out/sanitize/racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize/status.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -m gpu -q -x tests/test_gpu_csc_native.py tests/test_gpu_group.py -k "band_forms or detects_interior or group_matches or f64_bitexact" > gpurun_out/sanitize/synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/sanitize/status.txt
