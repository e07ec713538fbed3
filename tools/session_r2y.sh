bash tools/gpu_run.sh r2y all "" "" > gpurun_out/r2y_session.txt 2>&1
CFG=ds_v2_lite_decode ENVS="X=0|TG_EARLYMAX=0" bash tools/ab_env.sh > gpurun_out/r2y_ab.txt 2>&1
CFG=mixtral_decode ENVS="X=0|TG_EARLYMAX=0" bash tools/ab_env.sh >> gpurun_out/r2y_ab.txt 2>&1
python tools/trace_gemm.py --config ds_v2_lite_decode --warm 300 > gpurun_out/r2y_trace_ds.txt 2>&1
