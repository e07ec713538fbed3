mkdir -p gpurun_out
for ns in 4 8 2; do echo "== nsplit $ns"; TG_NSPLIT=$ns timeout 300 python tools/trace_gemm.py 2>&1 | grep -E "units|per-SM|kind"; TG_NSPLIT=$ns timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('bench', l['ms_per_step'], l['roofline']['per_kernel_ms'], l['clocks']['sm_mhz'])"; done > gpurun_out/nsplit.log 2>&1
cat gpurun_out/nsplit.log
