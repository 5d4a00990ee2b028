#!/bin/bash
# Device-checked build on the GPU box: compile the library with -DBD_CHECKS=1 (traps on the
# data-dependent indices, csrc/bd_common.cuh BD_CHECK) and run the GPU parity suites through it.
#   tools/checks_run.sh [OUTDIR]        (default gpurun_out/checks)
# A trap aborts the CUDA context, so every test after it fails: a green run means no check fired.
set -e
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/checks}
mkdir -p "$out"
lib=/tmp/libbilevel_b200_checks.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -prec-div=false -prec-sqrt=false -ftz=true -DBD_CHECKS=1 -o $lib paper_2212_02224_b200/csrc/bd_api.cu
set +e
BD_LIB_PATH=$lib python -m pytest -s -m gpu -q -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_cem.py tests/test_gpu_fleet.py tests/test_gpu_shapes.py \
  tests/test_gpu_random_parity.py tests/test_gpu_worlds.py tests/test_gpu_sim.py tests/test_gpu_cvae.py \
  tests/test_gpu_persistent.py tests/test_gpu_numpy_stream.py tests/test_gpu_spec_bilevel.py \
  > "$out/pytest_checks.log" 2>&1
rc=$?
fired=$(grep -c "BD_CHECK failed" "$out/pytest_checks.log")
{ echo "library: $lib (-DBD_CHECKS=1)"; echo "pytest rc: $rc"; echo "BD_CHECK failures: $fired";
  tail -3 "$out/pytest_checks.log"; } > "$out/summary.txt"
cat "$out/summary.txt"
exit $rc
