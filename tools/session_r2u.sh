bash tools/gpu_run.sh r2u all "" "" > gpurun_out/r2u_session.txt 2>&1
CFG=mixtral_decode ENVS="X=0|TG_NSPLIT=2|tree=ab_old" bash tools/ab_mg.sh > gpurun_out/r2u_n4.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 CFG=mixtral_decode ENVS="X=0|TG_NSPLIT=2|tree=ab_old" bash tools/ab_mg.sh > gpurun_out/r2u_n2.txt 2>&1
CFG=qwen_prefill ENVS="X=0|tree=ab_old" bash tools/ab_mg.sh > gpurun_out/r2u_n4q.txt 2>&1
