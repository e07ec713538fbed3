python paper_2601_01310_b200/build.py
timeout 900 python -m pytest tests -x -q -m gpu -k "not multi_gpu and not tile_modes" > gpurun_out/gpu_q.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/gpu_q.log
bash tools/gpu_ab2.sh 2>&1 | grep value
python tools/trace_gemm.py 2>&1 | grep "front kernel"
