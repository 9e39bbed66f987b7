# session 4: after the instruction diet of the fused passes (r1 / r2 / 2D): fast-path tests, then bench lines
timeout 1200 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_fast_policies.py tests/test_gpu_pyramid.py tests/test_gpu_complex64.py tests/test_gpu_graphs.py tests/test_gpu_goldens.py -x 2>&1 | tail -2
for a in "cfg2 fast" "cfg2 fast-complex64" "cfg1 fast" "cfg3 fast-complex64" "cfg5 fast-complex64" "cfg3 fast"; do set -- $a
  python bench.py --workload $1 --precision $2 --no-cpu-baseline --no-e2e > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); print('$1 $2', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d.get('fine_pass_ms',0),4))" || tail -3 gpurun_out/var.err
done
