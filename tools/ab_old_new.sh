# Same-box A/B: the round-start tree (ab_old/, built from 55d8680) against this tree under
# TG_LOCAL variants.  Prints "variant config us/call sm_mhz reasons".
python __graft_entry__.py > /dev/null 2>&1
CFGS=${CFGS:-"mixtral_decode qwen_prefill"}
VARS=${VARS:-"old 1 0 r c"}
for i in 1 2; do
 for v in $VARS; do
  for c in $CFGS; do
   if [ $v = old ]; then d=ab_old; unset TG_DEV; else d=.; export TG_DEV=$v; fi
   (cd $d && timeout 300 python bench.py --config $c --steps 300 --warmup 20 --no-cpu-baseline 2>/dev/null) | python -c "import json,sys; d=json.load(sys.stdin); print('$v $c', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
 done
done
