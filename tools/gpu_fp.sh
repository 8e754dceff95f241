# fused-pivot check: parity suites + large single-GPU + benches C1/C2/C3
set -x
mkdir -p gpurun_out
TAG=${TAG:-fp}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mps.py tests/test_gpu_tiled.py tests/test_gpu_cxx_dropin.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pt_fp_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_fp_$TAG.log
timeout 1500 python -m pytest tests/test_gpu_large.py -q -x --timeout 900 -p no:cacheprovider -k "single" > gpurun_out/pt_fp_large_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_fp_large_$TAG.log
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --steps 400 --warmup 20 --no-cpu-baseline --e2e-max-iter 2000 --no-reinversion > gpurun_out/bench_${c}_$TAG.log 2>&1; done
tail -n 3 gpurun_out/pt_fp_$TAG.log; tail -n 3 gpurun_out/pt_fp_large_$TAG.log
python - <<PY
import json
for c in ("c1", "c2", "c3"):
    try:
        l = json.loads(open(f"gpurun_out/bench_{c}_$TAG.log").read().strip().splitlines()[-1])
        r = l["roofline"]
        print(c, round(l["value"], 1), "it/s e2e", round(l["e2e"]["value"], 1), "frac", r["frac"], r["per_pivot"]["frac"],
              {k: (v["us_per_launch"], v.get("gbs")) for k, v in r["kernels"].items()})
    except Exception as e:
        print(c, "ERR", e)
PY
