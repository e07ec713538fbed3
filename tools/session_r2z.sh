python __graft_entry__.py > gpurun_out/r2z_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2z_smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rA > gpurun_out/r2z_tests.log 2>&1
tail -3 gpurun_out/r2z_tests.log
CFG=qwen_prefill ENVS="X=0|tree=ab_old|tree=ab_d7ff069|tree=ab_dd1d50e" bash tools/ab_mg.sh > gpurun_out/r2z_qwen4.txt 2>&1
