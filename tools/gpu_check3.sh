# GPU check: observer/dropin tests + large sharded parity at the deployment shard counts
set -x
mkdir -p gpurun_out
TAG=${TAG:-d}
make -s -C oracle dropin >/dev/null 2>&1 || true
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cxx_dropin.py -q -x --timeout 600 -p no:cacheprovider -k "observer or dropin" > gpurun_out/pt_obs_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_obs_$TAG.log
timeout 2400 python -m pytest tests/test_gpu_large.py -q --timeout 1500 -p no:cacheprovider -k "sharded and (c3_p200 or c5_p10 or c4_p20 or c2_full)" --durations=0 > gpurun_out/pt_large_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_large_$TAG.log
tail -5 gpurun_out/pt_obs_$TAG.log; tail -25 gpurun_out/pt_large_$TAG.log
