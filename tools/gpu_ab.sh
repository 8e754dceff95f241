mkdir -p gpurun_out
rm -f gpurun_out/ab.log
for args in "" "--no-profile" "--batch 16 --no-profile" "--batch 64 --no-profile" "--batch 64"; do
  echo "ARGS: $args" >> gpurun_out/ab.log
  timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline $args | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(l['value'],1), 'it/s', round(l['ms_per_step'],4),'ms')
for k,v in ((l.get('roofline') or {}).get('kernels') or {}).items(): print('   ',k, v['us_per_launch'], v['gbs'])
" >> gpurun_out/ab.log 2>&1
done
