# quick GPU check: parity subset + C3/C2 bench (no CPU baseline, bounded e2e)
set -x
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pt_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_$TAG.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --e2e-max-iter 400 > gpurun_out/bench_c3_$TAG.log 2>&1
timeout 300 python bench.py --config c2 --steps 200 --warmup 20 --no-cpu-baseline --e2e-max-iter 400 > gpurun_out/bench_c2_$TAG.log 2>&1
tail -2 gpurun_out/pt_$TAG.log
python - <<'PY'
import json, os
tag = os.environ.get("TAG", "q")
for c in ("c3", "c2"):
    try:
        l = json.loads(open(f"gpurun_out/bench_{c}_{tag}.log").read().strip().splitlines()[-1])
        print(c, round(l["value"], 1), "it/s", "frac", l["roofline"]["per_pivot"]["frac"],
              {k: (v["us_per_launch"], v.get("gbs", v.get("tflops"))) for k, v in l["roofline"]["kernels"].items()})
    except Exception as e:
        print(c, "ERR", e)
PY
