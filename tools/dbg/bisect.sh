# usage: bash tools/dbg/bisect.sh  — time C3 with each library under bisect_libs/ and the current one
cp paper_1803_04378_b200/_lib/liblpsg.so /tmp/cur_liblpsg.so
for lib in bisect_libs/*/liblpsg.so /tmp/cur_liblpsg.so; do
  cp $lib paper_1803_04378_b200/_lib/liblpsg.so
  touch paper_1803_04378_b200/_lib/liblpsg.so
  r=$(timeout 200 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --e2e-max-iter 10 --no-profile | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(l['value'],1))")
  echo "$lib: $r"
done
cp /tmp/cur_liblpsg.so paper_1803_04378_b200/_lib/liblpsg.so
