# session 4: lean exact regular top-down: bit-identity tests, then A/B against variants/prev.so
timeout 1200 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_exact_parity.py tests/test_gpu_goldens.py tests/test_gpu_multichannel.py tests/test_gpu_reference_ports.py tests/test_gpu_units.py tests/test_gpu_vcycles.py tests/test_gpu_headline.py -x 2>&1 | tail -2
for v in variants/prev.so base; do for w in cfg3 cfg5 cfg2; do
  if [ "$v" = base ]; then lib=""; else lib="TMG_LIB=$PWD/$v"; fi
  env $lib python bench.py --workload $w --precision exact --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); print('exact $w $v', round(d['value']/1e9,3), round(d['ms_per_step'],4))" || tail -3 gpurun_out/var.err
done; done
