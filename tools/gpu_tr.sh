mkdir -p gpurun_out
for c in mixtral_decode ds_v2_lite_decode; do echo "== $c"; timeout 300 python tools/trace_gemm.py --config $c 2>&1 | sed -n 1,6p; done > gpurun_out/tr.log 2>&1
cat gpurun_out/tr.log
