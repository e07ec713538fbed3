# Same-box A/B of environment variants on one config: ENVS="A=1 B=2|C=3" (| separates variants)
python __graft_entry__.py > /dev/null 2>&1
CFG=${CFG:-mixtral_decode}
IFS='|' read -ra V <<< "$ENVS"
for i in 1 2; do
 for v in "${V[@]}"; do
  (env $v timeout 300 python bench.py --config $CFG --steps 300 --warmup 20 --no-cpu-baseline 2>/dev/null) | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
 done
done
