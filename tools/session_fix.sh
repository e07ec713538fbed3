python __graft_entry__.py > /dev/null 2>&1
for i in 1 2 3; do
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "back_to_back or host_entry" > gpurun_out/fix_stress_$i.log 2>&1; tail -1 gpurun_out/fix_stress_$i.log
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rA > gpurun_out/fix_tests.log 2>&1; tail -1 gpurun_out/fix_tests.log
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fix_bench_ref.json 2> gpurun_out/fix_bench_ref.err
