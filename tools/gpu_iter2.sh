# parity + front trace + short bench (one GPU)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/iter.log
for c in mixtral_decode ds_v2_lite_decode qwen_prefill; do echo "== $c"; timeout 300 python tools/trace_gemm.py --config $c 2>&1 | sed -n 1,6p; done >> gpurun_out/iter.log 2>&1
timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('bench', l['ms_per_step'], l['roofline']['per_kernel_ms'], l['clocks'])" >> gpurun_out/iter.log 2>&1
cat gpurun_out/iter.log
