# Second end-of-round pass (after the lookahead changes): C4 bench line, the
# whole GPU suite and smoke().
set -x
mkdir -p gpurun_out
TAG=${TAG:-final2}
timeout 900 python bench.py --config c4 --steps 100 --warmup 3 --no-cpu-baseline --e2e-max-iter 300 > gpurun_out/bench_c4_$TAG.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -n 3 gpurun_out/pytest_gpu_$TAG.log
tail -n 2 gpurun_out/smoke_$TAG.log
