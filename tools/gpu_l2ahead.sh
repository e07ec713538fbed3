mkdir -p gpurun_out
for i in 1 2; do for v in 0 4 8 16; do
TG_L2AHEAD=$v timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('ahead=$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
done; done
