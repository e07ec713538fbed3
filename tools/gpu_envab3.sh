# env A/B/C on bench.py (same box, alternating, 2 rounds)
mkdir -p gpurun_out
for i in 1 2; do for e in "$@"; do
env $e timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$e', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done; done
