bash tools/gpu_run.sh r3c all "" "" > gpurun_out/r3c_session.txt 2>&1
python tools/trace_gemm.py --config qwen_prefill --W 4 --warm 50 > gpurun_out/r3c_trace_q.txt 2>&1
VARS="old 0" CFGS="qwen_prefill ds_v2_lite_decode" bash tools/ab_old_new.sh > gpurun_out/r3c_ab.txt 2>&1
