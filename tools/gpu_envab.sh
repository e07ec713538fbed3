# A/B of an env setting on bench.py (same box, alternating): gpu_envab.sh "VAR=a" "VAR=b" [bench args]
mkdir -p gpurun_out
A=$1; B=$2; shift 2
for i in 1 2; do for e in "$A" "$B"; do
env $e timeout 300 python bench.py --no-cpu-baseline --steps 1000 "$@" > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$e', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['roofline']['frac'])"
done; done
