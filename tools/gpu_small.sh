# chain-bound shapes: parity, C1/C2/C4 benches, per-GPU sharded shapes (pricing n=2000 / m=8000;
# forced h=8 update through the experiments library)
set -x
mkdir -p gpurun_out
TAG=${TAG:-sm}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_tiled.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pt_sm_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_sm_$TAG.log
timeout 1500 python -m pytest tests/test_gpu_large.py -q -x --timeout 900 -p no:cacheprovider -k "c2_full or c4_p20 or c3_p200" > gpurun_out/pt_sm_large_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_sm_large_$TAG.log
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 400 --warmup 20 --no-cpu-baseline --e2e-max-iter 2000 --no-reinversion > gpurun_out/bench_${c}_$TAG.log 2>&1; done
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --e2e-max-iter 300 --no-reinversion > gpurun_out/bench_c3_$TAG.log 2>&1
PYTHONPATH=. timeout 300 python tools/dbg/shape_probe.py 8000 2000 > gpurun_out/shape_price_$TAG.log 2>&1
python -c "from paper_1803_04378_b200 import build as b; b.build(experiments=True)" > /dev/null 2>&1
LPSG_EXPERIMENTS_LIB=1 LPSG_UPD_H=8 PYTHONPATH=. timeout 300 python tools/dbg/shape_probe.py 8000 16000 > gpurun_out/shape_upd8_$TAG.log 2>&1
tail -n 3 gpurun_out/pt_sm_$TAG.log; tail -n 3 gpurun_out/pt_sm_large_$TAG.log
cat gpurun_out/shape_price_$TAG.log gpurun_out/shape_upd8_$TAG.log | tail -4
python - <<PY
import json
for c in ("c1", "c2", "c3"):
    try:
        l = json.loads(open(f"gpurun_out/bench_{c}_$TAG.log").read().strip().splitlines()[-1])
        r = l["roofline"]
        print(c, round(l["value"], 1), "it/s", r["frac"], {k: (v["us_per_launch"], v.get("gbs")) for k, v in r["kernels"].items()})
    except Exception as e:
        print(c, "ERR", e)
PY
