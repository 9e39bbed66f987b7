#!/bin/bash
mkdir -p gpurun_out
TMG_LIB=$PWD/variants/rows2.so timeout 900 python -m pytest tests/test_gpu_goldens.py tests/test_gpu_headline.py tests/test_gpu_slabs.py tests/test_gpu_complex64.py tests/test_gpu_pyramid.py tests/test_gpu_fast_policies.py -m gpu -q -x -k "fast or headline or slabs or complex64 or single_launch or polic" --timeout 900 > gpurun_out/gputests_rows2.log 2>&1; tail -3 gpurun_out/gputests_rows2.log
timeout 900 bash scripts/variants.sh "cfg5 cfg3" "base variants/rows2.so" > gpurun_out/var.log 2>&1; cat gpurun_out/var.log
