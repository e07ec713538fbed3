set -x
python paper_2601_01310_b200/build.py
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "mixtral or ds_ or qwen" > gpurun_out/gpu_big.log 2>&1; echo big_rc=$?
tail -30 gpurun_out/gpu_big.log
timeout 600 python bench.py > gpurun_out/bench1.log 2>&1; echo bench_rc=$?
tail -5 gpurun_out/bench1.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
tail -5 gpurun_out/ncu_full.log
