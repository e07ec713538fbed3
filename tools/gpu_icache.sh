mkdir -p gpurun_out
( echo "== normal"; timeout 300 python tools/trace_gemm.py 2>&1 | sed -n 1,5p
  echo "== skip gemm"; TG_SKIP_GEMM=1 timeout 300 python tools/trace_gemm.py 2>&1 | sed -n 1,5p
  echo "== ds normal"; timeout 300 python tools/trace_gemm.py --config ds_v2_lite_decode 2>&1 | sed -n 1,5p
  echo "== ds skip gemm"; TG_SKIP_GEMM=1 timeout 300 python tools/trace_gemm.py --config ds_v2_lite_decode 2>&1 | sed -n 1,5p ) > gpurun_out/icache.log 2>&1
cat gpurun_out/icache.log
