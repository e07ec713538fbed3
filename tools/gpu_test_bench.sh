# full GPU test suite + default bench (no ncu)
python paper_2601_01310_b200/build.py
timeout 1200 python -m pytest tests -x -q -m gpu -s > gpurun_out/gpu_all.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|Error|tiny|mixtral|ds_v2|qwen" gpurun_out/gpu_all.log | tail -20
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -2 gpurun_out/bench.log
