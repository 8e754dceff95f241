for cfg in "X=1" "LPSG_NO_L2_HINT=1" "LPSG_UPD_COLS=16" "LPSG_UPD_COLS=16 LPSG_NO_L2_HINT=1" "LPSG_UPD_COLS=32 LPSG_UPD_STAGES=5"; do
  for c in c5 c3; do
  r=$(env $cfg timeout 200 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-max-iter 5 | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=l['roofline']['kernels']
print(round(l['value'],1), k['price']['us_per_launch'], k['update_ftran']['us_per_launch'])")
  echo "$c $cfg: $r"
  done
done
