python __graft_entry__.py > /dev/null 2>&1
for v in "X=0" "TG_LOCAL=0"; do
  echo "== $v"
  env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tests/mp_parity.py --config mixtral_decode --sample 16 2>/dev/null | grep -oE '"errors": .*'
done
