set -x
python paper_2601_01310_b200/build.py
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_router|k_rank|k_dispatch|k_combine" -s 20 -c 4 -o gpurun_out/prof_small python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_small.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "ds_ or qwen" > gpurun_out/gpu_big2.log 2>&1; echo big_rc=$?
tail -30 gpurun_out/gpu_big2.log
