# Multi-GPU session (gpurun --gpus N): torchrun parity tests, bench at N, NVLink counters.
G=$(python -c "import torch; print(torch.cuda.device_count())")
python __graft_entry__.py > gpurun_out/mg_build.log 2>&1
timeout 1500 python -m pytest tests/test_multi_gpu.py -q -p no:cacheprovider --timeout 900 -rA -s > gpurun_out/mg${G}_tests.log 2>&1
tail -3 gpurun_out/mg${G}_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $G --steps 500 --warmup 20 > gpurun_out/mg${G}_bench.json 2> gpurun_out/mg${G}_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $G --steps 100 --warmup 10 --config qwen_prefill > gpurun_out/mg${G}_bench_qwen.json 2> gpurun_out/mg${G}_bench_qwen.err
for c in qwen_prefill mixtral_decode; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29612 tools/nvlink_counters.py --config $c --W $((2*G)) > gpurun_out/mg${G}_nvlink_$c.json 2> gpurun_out/mg${G}_nvlink_$c.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29613 tools/trace_mp.py --config mixtral_decode > gpurun_out/mg${G}_trace_mixtral.jsonl 2> gpurun_out/mg${G}_trace.err
