CFGS=mixtral_decode ENVS="TG_NSPLIT=2|TG_NSPLIT=4" bash tools/ab_env.sh > gpurun_out/split_n1.txt 2>&1
CFG=mixtral_decode ENVS="TG_NSPLIT=2|TG_NSPLIT=4" bash tools/ab_mg.sh > gpurun_out/split_n2.txt 2>&1
