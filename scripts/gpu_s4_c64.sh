# session 4: complex64 in 2D: tests + bench lines (cfg2 / cfg1, complex128 beside complex64) + 2D regression tests
timeout 1300 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_complex64.py -s 2>&1 | grep -E "complex64|passed|failed" | tail -20
timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_fast_policies.py tests/test_gpu_pyramid.py tests/test_gpu_graphs.py -x 2>&1 | tail -2
mkdir -p gpurun_out/s4c
for w in cfg2 cfg1; do for p in fast fast-complex64; do
  python bench.py --workload $w --precision $p --no-cpu-baseline > gpurun_out/s4c/bench_${w}_$p.json 2> gpurun_out/s4c/bench_${w}_$p.err
  python -c "
import json; d=json.load(open('gpurun_out/s4c/bench_${w}_$p.json')); print('$w $p', round(d['value']/1e9,3), 'G', round(d['ms_per_step'],4), 'ms fine', round(d.get('fine_pass_ms',0),4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2))" || tail -3 gpurun_out/s4c/bench_${w}_$p.err
done; done
