# session 4: direct chi gather (order table instead of stored lists for interior kRegularChi vertices)
timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_amr.py tests/test_gpu_amr_fast.py tests/test_gpu_graphs.py -x 2>&1 | tail -3
for e in TMG_CHI_DIRECT=1 TMG_CHI_DIRECT=0; do for pr in fast exact; do
  env $e python bench.py --workload cfg4 --precision $pr --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('cfg4 $pr $e', round(d['value']/1e9,3), round(d['ms_per_step'],4))" || tail -3 gpurun_out/ab.err
done; done
