python paper_2601_01310_b200/build.py
G=$(python -c "import torch;print(torch.cuda.device_count())")
echo "GPUs: $G"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29555 tests/mp_parity.py --config tiny > gpurun_out/mp_tiny.log 2>&1; echo mp_tiny_rc=$?
tail -5 gpurun_out/mp_tiny.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29556 tests/mp_parity.py --config tiny --W $((2*G)) > gpurun_out/mp_tiny2.log 2>&1; echo mp_tiny2_rc=$?
tail -3 gpurun_out/mp_tiny2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29557 tests/mp_parity.py --config mixtral_decode --sample 16 > gpurun_out/mp_mix.log 2>&1; echo mp_mix_rc=$?
tail -3 gpurun_out/mp_mix.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr 127.0.0.1 --master-port 29558 bench.py --gpus $G > gpurun_out/bench_mg.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/bench_mg.log
