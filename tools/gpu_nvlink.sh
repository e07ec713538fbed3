python paper_2601_01310_b200/build.py
G=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29561 tools/nvlink_sweep.py --config qwen_prefill > gpurun_out/nvl_qwen_G$G.log 2>&1; echo rc=$?
grep "^{" gpurun_out/nvl_qwen_G$G.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29562 tools/nvlink_sweep.py --config mixtral_decode --tokens 256,1024,4096 > gpurun_out/nvl_mix_G$G.log 2>&1; echo rc=$?
grep "^{" gpurun_out/nvl_mix_G$G.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29563 bench.py --config qwen_prefill --steps 100 > gpurun_out/bench_qwen_G$G.log 2>&1; echo rc=$?
tail -1 gpurun_out/bench_qwen_G$G.log | cut -c1-300
