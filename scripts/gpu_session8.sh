#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
TMG_LIB=$PWD/variants/rows2ty4.so timeout 900 python -m pytest tests/test_gpu_goldens.py tests/test_gpu_headline.py tests/test_gpu_slabs.py tests/test_gpu_complex64.py -m gpu -q -x -k "fast or headline or slabs or complex64" --timeout 900 > gpurun_out/gputests_r2t4.log 2>&1; tail -3 gpurun_out/gputests_r2t4.log
timeout 1200 bash scripts/variants.sh "cfg5 cfg3" "base variants/rows2.so variants/rows2ty4.so variants/rows2ty4m3.so" > gpurun_out/var.log 2>&1; cat gpurun_out/var.log
