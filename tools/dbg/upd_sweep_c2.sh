for cfg in "8 32" "8 64" "8 128" "6 256" "4 512"; do
  set -- $cfg
  for c in c2 c1; do
  r=$(LPSG_UPD_STAGES=$1 LPSG_UPD_COLS=$2 timeout 120 python bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline --e2e-max-iter 10 | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=l['roofline']['kernels']
print(round(l['value'],1), k['update_ftran']['us_per_launch'], k['price']['us_per_launch'])")
  echo "$c S=$1 C=$2: $r"
  done
done
