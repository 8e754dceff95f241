# ncu evidence for the chain-bound small-m shapes: C2 k_price / k_update / k_pivot and the per-GPU
# pricing shape of an 8-way sharded C3 (m = 8000, n = 2000)
set -x
mkdir -p gpurun_out
TAG=${TAG:-c2}
for k in k_update k_price k_pivot; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 60 -c 1 -o gpurun_out/prof_c2_${k}_$TAG python bench.py --config c2 --steps 100 --warmup 20 --no-cpu-baseline --e2e-max-iter 5 --no-profile --no-reinversion > gpurun_out/ncu_c2_${k}_$TAG.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_price -s 30 -c 1 -o gpurun_out/prof_shape_price_$TAG env PYTHONPATH=. python tools/dbg/shape_probe.py 8000 2000 > gpurun_out/ncu_shape_$TAG.log 2>&1
ls gpurun_out/*$TAG*.ncu-rep
