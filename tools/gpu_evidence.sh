# evidence for profiles/: plain bench, ncu launch list of the same command, ncu --set full of k_gemm and k_front
python paper_2601_01310_b200/build.py
timeout 600 python bench.py > gpurun_out/bench_ev.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_ev.log | cut -c1-200
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_front" -s 10 -c 2 -o gpurun_out/prof_r01_final python bench.py --steps 5 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
