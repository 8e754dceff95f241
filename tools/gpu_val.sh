# validation after host-loop changes: parity + tiled + sharded + large singles + C3 driver-shaped bench
set -x
mkdir -p gpurun_out
TAG=${TAG:-v}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiled.py tests/test_gpu_sharded.py tests/test_gpu_reinvert.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pt_val_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_val_$TAG.log
timeout 1500 python -m pytest tests/test_gpu_large.py -q -x --timeout 900 -p no:cacheprovider -k "single and (c2_full or c3_p200 or c4_p20)" > gpurun_out/pt_val_large_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_val_large_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-reinversion --no-cpu-baseline > gpurun_out/bench_c3_drv_$TAG.log 2>&1
timeout 600 python bench.py --config c2 --steps 200 --warmup 20 --no-reinversion --no-cpu-baseline --e2e-max-iter 400 > gpurun_out/bench_c2_$TAG.log 2>&1
tail -n 2 gpurun_out/pt_val_$TAG.log; tail -n 2 gpurun_out/pt_val_large_$TAG.log
python - <<PY
import json
for f in ("c3_drv", "c2"):
    l = json.loads(open(f"gpurun_out/bench_{f}_$TAG.log").read().strip().splitlines()[-1])
    print(f, round(l["value"], 1), "e2e", round(l["e2e"]["value"], 1), "launches", l["gpu_launches"])
PY
