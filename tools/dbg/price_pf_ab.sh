# A/B of k_price's L2 warm-up prefetch under PDL (experiments library knob LPSG_PRICE_PF).
# Measured: C3 2933 -> 2948-2960 it/s with 8 stages; a T-tile prefetch in k_update cost 0.3-2.3 % (removed)
export LPSG_EXPERIMENTS_LIB=1
for cfg in c3 c2; do
for pf in "0 0" "8 0" "16 0" "0 0" "8 0" "16 0"; do
  set -- $pf
  LPSG_PRICE_PF=$1 timeout 300 python bench.py --config $cfg --steps 400 --warmup 20 --no-cpu-baseline --e2e-max-iter 30 --no-reinversion 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$cfg', '$1 $2', round(l['value'],1), {k:v['us_per_launch'] for k,v in l['roofline']['kernels'].items()})"
done; done
