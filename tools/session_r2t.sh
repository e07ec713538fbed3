bash tools/gpu_run.sh r2t all "" "mixtral_decode" > gpurun_out/r2t_session.txt 2>&1
VARS="old 0" CFGS="mixtral_decode ds_v2_lite_decode" bash tools/ab_old_new.sh > gpurun_out/r2t_ab.txt 2>&1
python tools/trace_gemm.py --config mixtral_decode --warm 300 > gpurun_out/r2t_trace_mix.txt 2>&1
