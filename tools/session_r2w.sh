bash tools/gpu_run.sh r2w all "" "" > gpurun_out/r2w_session.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/r2w_bench_N1.json 2> gpurun_out/r2w_bench_N1.err
timeout 600 $TR --nproc-per-node 4 --master-port 29651 bench.py --gpus 4 --steps 500 --warmup 20 > gpurun_out/r2w_bench_N4.json 2> gpurun_out/r2w_bench_N4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29652 bench.py --gpus 2 --steps 500 --warmup 20 > gpurun_out/r2w_bench_N2.json 2> gpurun_out/r2w_bench_N2.err
VARS="old 0" CFGS="mixtral_decode" bash tools/ab_old_new.sh > gpurun_out/r2w_ab.txt 2>&1
