# parity, then A/B (env applied to both libs): gpu_ab4.sh <rev> [env...]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
rev=$1; shift
for i in 1 2; do
for lib in "" "$PWD/ab_$rev.so"; do
env "$@" TG_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('lib=${lib:-new}', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
done; done
