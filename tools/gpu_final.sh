# round-end evidence on a 4-GPU box: bench lines (N = 1, 2, 4; other configs), multi-GPU parity, traces
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 600 python bench.py > gpurun_out/final/bench_mixtral_decode_N1.log 2>&1; tail -1 gpurun_out/final/bench_mixtral_decode_N1.log > gpurun_out/final/bench_mixtral_decode_N1.json
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n > gpurun_out/final/bench_N$n.log 2>&1
  grep '^{' gpurun_out/final/bench_N$n.log | tail -1 > gpurun_out/final/bench_mixtral_decode_N$n.json
done
for cfg in ds_v2_lite_decode qwen_prefill; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/final/b_$cfg.log 2>&1; tail -1 gpurun_out/final/b_$cfg.log > gpurun_out/final/bench_$cfg.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29912 bench.py --gpus 2 --config qwen_prefill --no-cpu-baseline > gpurun_out/final/bq2.log 2>&1
grep '^{' gpurun_out/final/bq2.log | tail -1 > gpurun_out/final/bench_qwen_prefill_N2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29913 tests/mp_parity.py --config mixtral_decode --sample 16 > gpurun_out/final/mp4.log 2>&1
grep '^{' gpurun_out/final/mp4.log | tail -1 > gpurun_out/final/mp_parity_mixtral_G4.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29914 tests/mp_parity.py --config tiny --W 8 > gpurun_out/final/mp4t.log 2>&1
grep '^{' gpurun_out/final/mp4t.log | tail -1 > gpurun_out/final/mp_parity_tiny_G4_W8.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29915 tests/mp_parity.py --config tiny --inflight-fail > gpurun_out/final/mp4f.log 2>&1
grep '^{' gpurun_out/final/mp4f.log | tail -1 > gpurun_out/final/mp_inflight_fail_tiny_G4.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29916 tools/trace_mp.py > gpurun_out/final/trace_mp4.log 2>&1
grep '^{' gpurun_out/final/trace_mp4.log > gpurun_out/final/trace_mp_mixtral_G4.jsonl
for f in gpurun_out/final/*.json; do echo "$f: $(cut -c1-160 $f)"; done
timeout 900 python bench.py --impl reference > gpurun_out/final/ref.log 2>&1; tail -1 gpurun_out/final/ref.log > gpurun_out/final/bench_reference_N1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29917 bench.py --impl reference --gpus 2 > gpurun_out/final/ref2.log 2>&1; echo "ref N2 rc=$?"; grep '^{' gpurun_out/final/ref2.log | tail -1 | cut -c1-120
