mkdir -p gpurun_out
for i in 1 2; do for m in 0 1 2; do
TG_DMODE=$m timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('dmode=$m', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done; done
for m in 0 1 2; do echo "dmode $m"; TG_DMODE=$m timeout 300 python tools/trace_gemm.py 2>&1 | grep -E "front kernel|gemm: CTA"; done
