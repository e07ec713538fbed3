mkdir -p gpurun_out
( echo "== default"; timeout 300 python tools/trace_gemm.py 2>&1 | sed -n 1,4p
  echo "== L2PF=0"; TG_L2PF=0 timeout 300 python tools/trace_gemm.py 2>&1 | sed -n 1,4p
  echo "== T=32"; timeout 300 python tools/trace_gemm.py --tokens 32 2>&1 | sed -n 1,4p
  echo "== T=2048"; timeout 300 python tools/trace_gemm.py --tokens 2048 2>&1 | sed -n 1,4p ) > gpurun_out/front2.log 2>&1
cat gpurun_out/front2.log
