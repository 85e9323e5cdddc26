mkdir -p gpurun_out
for i in 1 2 3; do
  python bench.py --no-cpu-baseline > gpurun_out/e2e_def_$i.json 2>/dev/null
  CUDA_DEVICE_MAX_CONNECTIONS=32 python bench.py --no-cpu-baseline > gpurun_out/e2e_c32_$i.json 2>/dev/null
done
for f in gpurun_out/e2e_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['e2e']['value'],1), d['e2e']['ms_per_step'])"; done
