python __graft_entry__.py > /dev/null 2>&1
VARS="old 0" bash tools/ab_old_new.sh
python tools/trace_gemm.py --config mixtral_decode --warm 300 > gpurun_out/ab7_trace_mix.txt 2>&1
python tools/trace_gemm.py --config qwen_prefill --W 4 --warm 50 > gpurun_out/ab7_trace_q.txt 2>&1
