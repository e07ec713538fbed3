# Round-end evidence on one GPU: the default bench line, the ncu launch list of the same command,
# and one ncu --set full capture of k_layer at Mixtral decode and at the Qwen-shaped prefill
# (each ncu pass only after its command ran clean without ncu).  TAG=r02 by default.
TAG=${TAG:-r02}
python __graft_entry__.py > gpurun_out/${TAG}_fin_build.log 2>&1 || exit 1
python bench.py > gpurun_out/${TAG}_fin_bench_default.json 2> gpurun_out/${TAG}_fin_bench_default.err
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_fin_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_fin_launches.csv $CMD > gpurun_out/${TAG}_fin_ncu_launch.log 2>&1
for c in mixtral_decode qwen_prefill; do
  CMDC="python bench.py --config $c --steps 3 --warmup 10 --no-cpu-baseline"
  $CMDC > gpurun_out/${TAG}_fin_plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_layer -s 11 -c 1 \
      -o gpurun_out/${TAG}_fin_ncu_$c $CMDC > gpurun_out/${TAG}_fin_ncu_$c.log 2>&1
  ncu -i gpurun_out/${TAG}_fin_ncu_$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_fin_ncu_raw_$c.csv 2>/dev/null
done
