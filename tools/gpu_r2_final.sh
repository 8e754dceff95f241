# Round-2 evidence on one B200: C3 both arms (driver shape and default), C1/C2/C4/C5 benches,
# ncu launch list + full captures of the C3 kernels, the whole GPU suite and smoke().
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2f}
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-reinversion > gpurun_out/bench_c3_drv_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_c3_ref_$TAG.log 2>&1
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c1_$TAG.log 2>&1
timeout 300 python bench.py --config c2 --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.log 2>&1
timeout 900 python bench.py --config c4 --steps 60 --warmup 3 --no-cpu-baseline --e2e-max-iter 30 > gpurun_out/bench_c4_$TAG.log 2>&1
timeout 900 python bench.py --config c5 --steps 30 --warmup 5 --e2e-max-iter 40 > gpurun_out/bench_c5_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 100 --warmup 20 --no-cpu-baseline --e2e-max-iter 10 --no-profile --no-reinversion > /dev/null 2>&1
for k in k_update k_price k_pivot; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 60 --warmup 20 --no-cpu-baseline --e2e-max-iter 5 --no-profile --no-reinversion > gpurun_out/ncu_${k}_$TAG.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_la_screen|k_la_probe$" -s 2 -c 2 -o gpurun_out/prof_c4_$TAG python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --e2e-max-iter 2 --no-profile --no-reinversion > gpurun_out/ncu_c4_$TAG.log 2>&1
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 --durations=25 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -n 4 gpurun_out/pytest_gpu_$TAG.log; tail -n 2 gpurun_out/smoke_$TAG.log
python - <<PY
import json
for f in ("c3", "c3_drv", "c3_ref", "c1", "c2", "c4", "c5"):
    try:
        l = json.loads(open(f"gpurun_out/bench_{f}_$TAG.log").read().strip().splitlines()[-1])
        r = l.get("roofline") or {}
        print(f, round(l["value"], 2), "e2e", round(l["e2e"]["value"], 2), "frac", r.get("frac"), "cpu", (l.get("cpu_baseline") or {}).get("value"), "tto", (l.get("time_to_optimal") or {}).get("status"), (l.get("time_to_optimal_reinversion") or {}).get("status"))
    except Exception as e:
        print(f, "ERR", e)
PY
