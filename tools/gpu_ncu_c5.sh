# ncu --set full of C5's k_update and k_price (one launch each, after warm-up)
mkdir -p gpurun_out
TAG=${TAG:-c5}
for k in k_update k_price; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 1 -o gpurun_out/prof_c5_${k}_$TAG python bench.py --config c5 --steps 10 --warmup 5 --no-cpu-baseline --e2e-max-iter 2 --no-profile --no-reinversion > gpurun_out/ncu_c5_${k}_$TAG.log 2>&1
done
ls -la gpurun_out/prof_c5_*_$TAG*
