# session 4: A/B of compile-time variants of the adaptive level passes at cfg4 (fast), + parity of the class-sum stencil
mkdir -p gpurun_out/s4
bash scripts/variants.sh "cfg4" "base variants/cs.so variants/cs4.so variants/cs2.so variants/td4.so variants/td2.so"
TMG_LIB=$PWD/variants/cs.so timeout 600 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_amr_fast.py 2>&1 | tail -3
