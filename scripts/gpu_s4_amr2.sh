# session 4: lean static top-down path + multiply-high unflat in the adaptive passes: parity, then A/B against variants/prev.so
timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_amr.py tests/test_gpu_amr_fast.py tests/test_gpu_graphs.py tests/test_gpu_dynamic.py -x 2>&1 | tail -2
timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_goldens.py -k "cfg4 or amr" 2>&1 | tail -2
bash scripts/variants.sh "cfg4" "variants/prev.so base"
for v in variants/prev.so base; do
  if [ "$v" = base ]; then lib=""; else lib="TMG_LIB=$PWD/$v"; fi
  env $lib python bench.py --workload cfg4 --precision exact --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); print('cfg4 exact $v', round(d['value']/1e9,3), round(d['ms_per_step'],4))" || tail -3 gpurun_out/var.err
done
