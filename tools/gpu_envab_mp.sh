# env A/B at N = 1 and N = n: gpu_envab_mp.sh n "VAR=a" "VAR=b"
n=$1; A=$2; B=$3
mkdir -p gpurun_out
for i in 1 2; do for e in "$A" "$B"; do
env $e timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('N=1 $e', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
env $e timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$i bench.py --gpus $n --no-cpu-baseline > gpurun_out/abn.log 2>&1
python -c "
import json; d=json.loads([l for l in open('gpurun_out/abn.log').read().strip().splitlines() if l.startswith('{')][-1])
print('N=$n $e', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/abn.log
done; done
