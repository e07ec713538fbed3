# ncu --set full of k_layer at the Qwen-shaped prefill (one GPU), after the same command ran clean
python __graft_entry__.py > /dev/null 2>&1
CMD="python bench.py --config qwen_prefill --steps 3 --warmup 10 --no-cpu-baseline"
$CMD > gpurun_out/ncu_q_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_layer -s 11 -c 1 -o gpurun_out/r2_ncu_qwen $CMD > gpurun_out/ncu_q.log 2>&1
ncu -i gpurun_out/r2_ncu_qwen.ncu-rep --page raw --csv > gpurun_out/r2_ncu_qwen_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_ncu_qwen.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_ncu_qwen_src.csv 2>/dev/null
$CMD > gpurun_out/ncu_q_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 11 -c 5 --csv --log-file gpurun_out/r2_launches_qwen.csv $CMD > /dev/null 2>&1
