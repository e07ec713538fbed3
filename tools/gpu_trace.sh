python paper_2601_01310_b200/build.py
mkdir -p gpurun_out
timeout 300 python tools/trace_gemm.py 2>&1 | tail -12
timeout 300 python tools/trace_gemm.py --config qwen_prefill --W 1 2>&1 | tail -12
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_router|k_rank|k_dispatch|k_combine" -s 20 -c 4 -o gpurun_out/prof_small2 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1; echo ncu_rc=$?
