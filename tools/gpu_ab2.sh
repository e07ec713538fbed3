
for i in 1; do
for lib in ab_HEAD.so paper_2601_01310_b200/libtarragon.so; do
for c in mixtral_decode ds_v2_lite_decode; do
TG_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config $c --no-cpu-baseline --steps 200 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$lib $c', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in d['roofline']['per_kernel_ms'].items()})"
done; done; done
