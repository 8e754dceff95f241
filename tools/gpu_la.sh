# C4 lookahead: tie parity (small + large), C4 bench, ncu captures of both lookahead GEMMs
set -x
mkdir -p gpurun_out
TAG=${TAG:-la}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x --timeout 600 -p no:cacheprovider -k "f2 or beale or lookahead or netlib or bounded" > gpurun_out/pt_la_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_la_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_tiled.py -q --timeout 900 -p no:cacheprovider -k "c4 or tiled" > gpurun_out/pt_la_large_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_la_large_$TAG.log
timeout 900 python bench.py --config c4 --steps 60 --warmup 3 --no-cpu-baseline --e2e-max-iter 30 --no-reinversion > gpurun_out/bench_c4_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_la_gemm|k_la_screen|k_la_probe" -s 0 -c 12 -o gpurun_out/prof_la_$TAG python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --e2e-max-iter 2 --no-profile --no-reinversion > gpurun_out/ncu_la_$TAG.log 2>&1
tail -n 3 gpurun_out/pt_la_$TAG.log; tail -n 3 gpurun_out/pt_la_large_$TAG.log
python - <<PY
import json
l = json.loads(open("gpurun_out/bench_c4_$TAG.log").read().strip().splitlines()[-1])
r = l["roofline"]
print("c4", round(l["value"], 2), "it/s", r["bound"], r["kernel"], r["achieved"], r["peak"], r["frac"])
print({k: (v["us_per_launch"], v.get("tflops"), v.get("gbs")) for k, v in r["kernels"].items()})
PY
ls -la gpurun_out/prof_la_$TAG* 
