# Same-box A/B of environment variants under torchrun (gpurun --gpus G): CFG=..., ENVS="A=1|B=2";
# the variant "old" runs the tree in ab_r1/, "tree=DIR" the tree in DIR/ (builds of other revisions)
python __graft_entry__.py > /dev/null 2>&1
G=$(python -c "import torch; print(torch.cuda.device_count())")
CFG=${CFG:-qwen_prefill}
IFS='|' read -ra V <<< "$ENVS"
for i in 1 2; do
 for v in "${V[@]}"; do
  d=.; ev=$v; [ "$v" = old ] && { d=ab_r1; ev=X=0; }
  case "$v" in tree=*) d=${v#tree=}; ev=X=0;; esac
  (cd $d && env $ev timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29630 bench.py --gpus $G --config $CFG --steps 200 --warmup 20 --no-cpu-baseline 2>/dev/null) | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$v', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
 done
done
