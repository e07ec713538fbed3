python __graft_entry__.py > gpurun_out/fin_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/fin_smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rA > gpurun_out/fin_tests.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python bench.py > gpurun_out/fin_bench_default.json 2> gpurun_out/fin_bench_default.err
timeout 600 $TR --nproc-per-node 4 --master-port 29661 bench.py --gpus 4 --steps 500 --warmup 20 > gpurun_out/fin_bench_N4.json 2> gpurun_out/fin_bench_N4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29662 bench.py --gpus 2 --steps 500 --warmup 20 > gpurun_out/fin_bench_N2.json 2> gpurun_out/fin_bench_N2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29663 bench.py --gpus 4 --steps 100 --warmup 10 --config qwen_prefill > gpurun_out/fin_bench_qwen_N4.json 2> gpurun_out/fin_bench_qwen_N4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
