set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c3.log 2>&1
tail -3 gpurun_out/*.log
