mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 8 -c 2 -o gpurun_out/prof_update_$TAG python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_update_$TAG.log 2>&1
