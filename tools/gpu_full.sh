# Full solves (time to the final status) at C4 and C5 on one B200, parity mode and reinversion mode
set -x
mkdir -p gpurun_out
TAG=${TAG:-full}
timeout 2400 python bench.py --config c5 --steps 30 --warmup 5 --e2e-max-iter 0 > gpurun_out/bench_c5_full_$TAG.log 2>&1
timeout 2400 python bench.py --config c4 --steps 30 --warmup 3 --e2e-max-iter 0 --no-cpu-baseline > gpurun_out/bench_c4_full_$TAG.log 2>&1
python - <<PY
import json
for c in ("c5_full", "c4_full"):
    try:
        l = json.loads(open(f"gpurun_out/bench_{c}_$TAG.log").read().strip().splitlines()[-1])
        print(c, l["value"], l["time_to_optimal"], l.get("time_to_optimal_reinversion"))
    except Exception as e:
        print(c, "ERR", e, open(f"gpurun_out/bench_{c}_$TAG.log").read()[-1500:])
PY
