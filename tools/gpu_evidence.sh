# evidence for profiles/ (call A): plain bench, then the ncu launch list of a short bench command
# (run first without ncu)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_ev.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_ev.log | cut -c1-300
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
