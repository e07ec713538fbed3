# front-kernel breakdown + bench + L2 prefetch sweep (one GPU)
mkdir -p gpurun_out
for c in mixtral_decode ds_v2_lite_decode; do echo "== $c"; timeout 300 python tools/trace_gemm.py --config $c 2>&1 | head -8; done > gpurun_out/trace.log 2>&1
timeout 400 python -X faulthandler bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/trace.log
for pf in 0 25000000 50000000 80000000 110000000; do echo "L2PF=$pf" >> gpurun_out/trace.log; TG_L2PF=$pf timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['roofline']['per_kernel_ms'], l['clocks'])" >> gpurun_out/trace.log 2>&1; done
cat gpurun_out/trace.log; tail -2 gpurun_out/bench.log
