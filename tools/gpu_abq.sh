# parity, then A/B on the prefill and decode configs vs ab_<rev>.so
rev=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do for cfg in qwen_prefill mixtral_decode ds_v2_lite_decode; do for lib in "" "$PWD/ab_$rev.so"; do
TG_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 300 > gpurun_out/abq.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/abq.log').read().strip().splitlines()[-1])
print('$cfg lib=${lib:-new}', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/abq.log
done; done; done
