# GPU check: parity + sharded + mps + nccl suites, then C3 both bench arms (driver-shaped)
set -x
mkdir -p gpurun_out
TAG=${TAG:-c}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_mps.py tests/test_gpu_nccl.py tests/test_gpu_cxx_dropin.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pt_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_c3_ref_$TAG.log 2>&1
tail -3 gpurun_out/pt_$TAG.log
tail -c 600 gpurun_out/bench_c3_$TAG.log; echo; tail -c 400 gpurun_out/bench_c3_ref_$TAG.log
