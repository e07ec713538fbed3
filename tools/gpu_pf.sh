python paper_2601_01310_b200/build.py
for i in 1 2; do for pf in 0 50000000 100000000; do
TG_L2PF=$pf timeout 300 python bench.py --no-cpu-baseline --steps 400 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('L2PF=$pf', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in d['roofline']['per_kernel_ms'].items()})"
done; done
