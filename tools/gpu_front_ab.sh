rev=$1
for i in 1 2; do for lib in "" "$PWD/ab_$rev.so"; do
echo "lib=${lib:-new}"; TG_LIB_PATH=$lib timeout 300 python tools/trace_gemm.py --config qwen_prefill --warm 100 2>&1 | grep -E "front phases|P1 finish|gemm:"
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
bash tools/gpu_abq.sh $rev 2>&1 | grep -E "lib="
