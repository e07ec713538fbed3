# A/B of the working tree's libtarragon vs ab_$1.so (same box, alternating)
mkdir -p gpurun_out
for i in 1 2 3; do
for lib in "" "$PWD/ab_$1.so"; do
TG_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 1000 ${@:2} > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('lib=${lib:-new}', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['gpu_launches'])"
done; done
