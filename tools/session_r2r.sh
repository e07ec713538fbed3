bash tools/gpu_run.sh r2r all "" "" > gpurun_out/r2r_session.txt 2>&1
VARS="old 0" CFGS="mixtral_decode ds_v2_lite_decode qwen_prefill" bash tools/ab_old_new.sh > gpurun_out/r2r_ab.txt 2>&1
CFG=mixtral_decode ENVS="X=0" bash tools/ab_mg.sh > gpurun_out/r2r_mg.txt 2>&1
CFG=qwen_prefill ENVS="X=0" bash tools/ab_mg.sh >> gpurun_out/r2r_mg.txt 2>&1
CFG=ds_v2_lite_decode ENVS="X=0" bash tools/ab_mg.sh >> gpurun_out/r2r_mg.txt 2>&1
