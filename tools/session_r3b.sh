bash tools/gpu_run.sh r3b all "" "" > gpurun_out/r3b_session.txt 2>&1
VARS="old 0" CFGS="mixtral_decode ds_v2_lite_decode qwen_prefill" bash tools/ab_old_new.sh > gpurun_out/r3b_ab.txt 2>&1
python tools/trace_gemm.py --config mixtral_decode --warm 300 > gpurun_out/r3b_trace_mix.txt 2>&1
python tools/trace_gemm.py --config qwen_prefill --W 4 --warm 50 > gpurun_out/r3b_trace_q.txt 2>&1
