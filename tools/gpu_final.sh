# End-of-round evidence on one B200: the profile set (benches C1-C3 + ncu launch
# list + full captures), C4/C5 benches, the whole GPU test suite and smoke().
set -x
mkdir -p gpurun_out
TAG=${TAG:-final}
TAG=$TAG bash tools/gpu_profile.sh
timeout 900 python bench.py --config c4 --steps 100 --warmup 3 --no-cpu-baseline --e2e-max-iter 300 > gpurun_out/bench_c4_$TAG.log 2>&1
timeout 900 python bench.py --config c5 --steps 30 --warmup 5 --e2e-max-iter 40 > gpurun_out/bench_c5_$TAG.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log gpurun_out/smoke_$TAG.log
