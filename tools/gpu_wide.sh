python paper_2601_01310_b200/build.py
for w in 0 1; do echo "TG_WIDE=$w"; TG_WIDE=$w timeout 300 python tools/trace_gemm.py --config qwen_prefill 2>&1 | grep -E "units|per-SM|kind|gemm:"; done
