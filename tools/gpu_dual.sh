python paper_2601_01310_b200/build.py
timeout 1200 python -m pytest tests -x -q -m gpu -k "not multi_gpu" > gpurun_out/gpu_all.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/gpu_all.log
bash tools/gpu_ab2.sh 2>&1 | grep value
TG_G2DUAL=1 timeout 300 python tools/trace_gemm.py --config qwen_prefill 2>&1 | grep -E "units|per-SM|kind"
