# evidence for profiles/ (call B): ncu --set full of two k_layer launches (command first run without ncu)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tiny.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_layer" -s 10 -c 2 -o gpurun_out/prof_${1:-r01_fused} python bench.py --steps 5 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
