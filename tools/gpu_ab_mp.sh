# A/B of the working tree vs ab_<rev>.so at N in the list (default "1 4"), same box, 2 rounds
rev=$1; NS=${2:-"1 4"}
mkdir -p gpurun_out
for i in 1 2; do
for lib in "" "$PWD/ab_$rev.so"; do
for n in $NS; do
if [ $n = 1 ]; then
TG_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/abn.log 2>&1
else
TG_LIB_PATH=$lib timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 298$i$n bench.py --gpus $n --no-cpu-baseline > gpurun_out/abn.log 2>&1
fi
python -c "
import json; d=json.loads([l for l in open('gpurun_out/abn.log').read().strip().splitlines() if l.startswith('{')][-1])
print('N=$n lib=${lib:-new}', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/abn.log
done; done; done
