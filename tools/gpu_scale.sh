# bench at N = 1, 2, 4 on one box (the driver's scaling runs), plus per-rank traces at N = 2, 4
mkdir -p gpurun_out
G=$(python -c "import torch; print(torch.cuda.device_count())")
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/scale_1.log 2>&1; tail -1 gpurun_out/scale_1.log | cut -c1-200
for n in ${NS:-2 4}; do
  [ $n -le $G ] || continue
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n > gpurun_out/scale_$n.log 2>&1
  grep '^{' gpurun_out/scale_$n.log | tail -1 | cut -c1-200
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n tools/trace_mp.py > gpurun_out/trace_mp_$n.log 2>&1
  grep '^{' gpurun_out/trace_mp_$n.log
done
