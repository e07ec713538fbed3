python paper_2601_01310_b200/build.py
for c in qwen_prefill ds_v2_lite_decode; do
timeout 600 python bench.py --config $c --no-cpu-baseline --steps 100 > gpurun_out/bench_$c.log 2>&1; echo $c rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1])
print('$c', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'gemm frac', round(d['roofline']['frac'],3), {k: round(v*1000,1) for k,v in d['roofline']['per_kernel_ms'].items()})"
done
timeout 300 python tools/trace_gemm.py --config qwen_prefill 2>&1 | tail -8
for w in failover flip shadow; do timeout 600 python tools/protocols.py --which $w > gpurun_out/proto_$w.log 2>&1; echo $w rc=$?; tail -1 gpurun_out/proto_$w.log; done
