bash tools/gpu_run.sh r2v all "" "" > gpurun_out/r2v_session.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29641 bench.py --gpus 4 --steps 500 --warmup 20 > gpurun_out/r2v_bench_N4.json 2> gpurun_out/r2v_bench_N4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29642 bench.py --gpus 4 --steps 100 --warmup 10 --config qwen_prefill > gpurun_out/r2v_bench_qwen_N4.json 2> gpurun_out/r2v_bench_qwen_N4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29643 bench.py --gpus 2 --steps 500 --warmup 20 > gpurun_out/r2v_bench_N2.json 2> gpurun_out/r2v_bench_N2.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29644 bench.py --gpus 2 --steps 100 --warmup 10 --config qwen_prefill > gpurun_out/r2v_bench_qwen_N2.json 2> gpurun_out/r2v_bench_qwen_N2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29645 tools/trace_mp.py --config mixtral_decode > gpurun_out/r2v_trace_mp4.jsonl 2> gpurun_out/r2v_trace_mp4.err
CFG=ds_v2_lite_decode ENVS="X=0|TG_LAYOUT=8192" bash tools/ab_env.sh > gpurun_out/r2v_ds.txt 2>&1
