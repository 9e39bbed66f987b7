# session 4: A/B of the fused-3D-pass phase-B task map (bank conflicts)
mkdir -p gpurun_out/s4
TMG_LIB=$PWD/variants/tm.so timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_fast_policies.py tests/test_gpu_pyramid.py -x 2>&1 | tail -2
bash scripts/variants.sh "cfg3 cfg5" "base variants/tm.so"
