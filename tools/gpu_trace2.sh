python paper_2601_01310_b200/build.py
for p in 1 0; do echo "PDL=$p"; TG_PDL=$p timeout 300 python tools/trace_gemm.py 2>&1 | grep -E "front|gemm:|router"
TG_PDL=$p timeout 300 python tools/trace_gemm.py --config qwen_prefill 2>&1 | grep -E "front|gemm:|router"; done
