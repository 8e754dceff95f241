# Case 2 (tiled) parity + C4 lookahead check
set -x
mkdir -p gpurun_out
TAG=${TAG:-t}
timeout 1500 python -m pytest tests/test_gpu_tiled.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pt_tiled_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_tiled_$TAG.log
tail -n 25 gpurun_out/pt_tiled_$TAG.log
TAG=$TAG bash tools/gpu_la.sh
