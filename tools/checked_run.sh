#!/bin/bash
# The LG_CHECKS build (device-side shared-memory bounds checks, trap on
# violation) over the sanitizer cases and the GPU parity tests: the stand-in
# for compute-sanitizer, which is closed on this GPU pool.
#   nvcc ... -DLG_CHECKS -o variants/checked.so; bash tools/checked_run.sh
export LG_LIB_PATH=variants/checked.so
timeout 600 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo "cases rc=$?"; tail -2 gpurun_out/checked_cases.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_reference_semantics.py tests/test_gpu_chain.py tests/test_gpu_trunk.py -m gpu -q > gpurun_out/checked_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/checked_tests.log
