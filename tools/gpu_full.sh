# full single-GPU test suite + benches of all single-GPU configs
python paper_2601_01310_b200/build.py
timeout 1200 python -m pytest tests -x -q -m gpu -s > gpurun_out/gpu_all.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|Error|^tiny|mixtral_decode \{|ds_v2|qwen_prefill \{" gpurun_out/gpu_all.log | cut -c1-400 | tail -12
for c in mixtral_decode qwen_prefill ds_v2_lite_decode; do
timeout 600 python bench.py --config $c --no-cpu-baseline --steps 200 > gpurun_out/bench_$c.log 2>&1; echo $c rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1])
print('$c', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'gemm frac', round(d['roofline']['frac'],3), {k: round(v*1000,1) for k,v in d['roofline']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
timeout 300 python tools/trace_gemm.py --config qwen_prefill 2>&1 | grep -E "front|gemm:"
timeout 300 python tools/trace_gemm.py 2>&1 | grep -E "front|gemm:"
