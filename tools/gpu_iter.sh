# quick iteration: tiny+mixtral parity, trace, bench
python paper_2601_01310_b200/build.py
timeout 600 python -m pytest tests -x -q -m gpu -k "tiny or ragged or flip or mixtral or ties or empty" > gpurun_out/gpu_iter.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/gpu_iter.log
timeout 300 python tools/trace_gemm.py 2>&1 | tail -8
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'gemm frac', round(d['roofline']['frac'],3), {k: round(v*1000,1) for k,v in d['roofline']['per_kernel_ms'].items()}, d['clocks'])"
