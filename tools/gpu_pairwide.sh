rev=$1
mkdir -p gpurun_out
TG_WIDE=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "qwen or tiny_parity" 2>&1 | tail -1
for i in 1 2; do
for v in "TG_WIDE=1" "TG_WIDE=0"; do
env $v timeout 300 python bench.py --config qwen_prefill --no-cpu-baseline --steps 300 > gpurun_out/pw.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/pw.log').read().strip().splitlines()[-1]); print('pair $v', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
TG_LIB_PATH=$PWD/ab_$rev.so timeout 300 python bench.py --config qwen_prefill --no-cpu-baseline --steps 300 > gpurun_out/pw.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/pw.log').read().strip().splitlines()[-1]); print('product', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
