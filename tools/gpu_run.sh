# One parametrised GPU session script (replaces the per-experiment gpu_*.sh one-offs).
#   bash tools/gpu_run.sh TAG "pytest -k expression ('' = no tests, 'all' = every gpu test)" "bench configs" [trace configs]
# Writes gpurun_out/TAG_*.{log,json,txt}.
TAG=$1; SEL=$2; BENCH=$3; TRACE=$4
python __graft_entry__.py > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
if [ "$SEL" = all ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rA -s > gpurun_out/${TAG}_tests.log 2>&1
  tail -3 gpurun_out/${TAG}_tests.log
elif [ -n "$SEL" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rA -k "$SEL" -s > gpurun_out/${TAG}_tests.log 2>&1
  tail -3 gpurun_out/${TAG}_tests.log
fi
for c in $BENCH; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  cat gpurun_out/${TAG}_bench_$c.json | python -c "import json,sys; d=json.load(sys.stdin); print('$c', round(d['ms_per_step']*1e3,1), 'us', d['roofline']['bound'], round(d['roofline']['frac'],3), d['clocks'])" 2>/dev/null
done
for c in $TRACE; do
  W=1; [ $c = qwen_prefill ] && W=4
  timeout 300 python tools/trace_gemm.py --config $c --W $W > gpurun_out/${TAG}_trace_$c.txt 2>&1
done
