# A/B: PDL on/off, 3 alternating runs each
python paper_2601_01310_b200/build.py
for i in 1 2 3; do
for p in 0 1; do
TG_PDL=$p timeout 300 python bench.py --no-cpu-baseline --steps 600 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('PDL=$p', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in d['roofline']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done; done
