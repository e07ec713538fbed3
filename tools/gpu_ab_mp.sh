# A/B of the working tree vs ab_<rev>.so at N = 1 and N = $2 (default 4), same box
rev=$1; n=${2:-4}
mkdir -p gpurun_out
for i in 1 2; do
for lib in "" "$PWD/ab_$rev.so"; do
TG_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/ab.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('N=1 lib=${lib:-new}', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
TG_LIB_PATH=$lib timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$i bench.py --gpus $n --no-cpu-baseline > gpurun_out/abn.log 2>&1
python -c "
import json; d=json.loads([l for l in open('gpurun_out/abn.log').read().strip().splitlines() if l.startswith('{')][-1])
print('N=$n lib=${lib:-new}', 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/abn.log
done; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29799 tools/trace_mp.py 2>&1 | grep "^{"
