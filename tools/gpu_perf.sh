# GPU round trip: parity tests, benches, ncu launch list + one full capture per hot kernel.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r}
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c1_$TAG.log 2>&1
timeout 300 python bench.py --config c2 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 20 ${BENCH_EXTRA} > gpurun_out/bench_c3_$TAG.log 2>&1
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 8 -c 1 -o gpurun_out/prof_update_$TAG python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_update_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_price -s 8 -c 1 -o gpurun_out/prof_price_$TAG python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_price_$TAG.log 2>&1
fi
tail -n 3 gpurun_out/pytest_gpu_$TAG.log
