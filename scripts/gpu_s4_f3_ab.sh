# session 4: A/B of a fused-3D-pass change: variants/prev.so (previous build) against the in-tree library
mkdir -p gpurun_out/s4
timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_fast_policies.py tests/test_gpu_pyramid.py tests/test_gpu_headline.py tests/test_gpu_slabs.py -x 2>&1 | tail -2
bash scripts/variants.sh "cfg3 cfg5" "variants/prev.so base"
for v in variants/prev.so base; do
  if [ "$v" = base ]; then lib=""; else lib="TMG_LIB=$PWD/$v"; fi
  env $lib python bench.py --steps 400 --no-cpu-baseline --no-e2e > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); print('cfg5 x400 $v', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('fine_pass_ms',0),4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/var.err
done
