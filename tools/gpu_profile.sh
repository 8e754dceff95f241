# Round profile: benches (C3 with CPU baseline, C1, C2) + ncu launch list + full captures.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r}
[ -z "$NCU_ONLY" ] && timeout 600 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1
[ -z "$NCU_ONLY" ] && timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c1_$TAG.log 2>&1
[ -z "$NCU_ONLY" ] && timeout 300 python bench.py --config c2 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.log 2>&1
# launch list: one 100-pivot window (pipelined batches leave a few no-op launches at each stop)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 100 --warmup 20 --no-cpu-baseline --e2e-max-iter 10 --no-profile > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 40 -c 1 -o gpurun_out/prof_update_$TAG python bench.py --steps 60 --warmup 20 --no-cpu-baseline --e2e-max-iter 5 --no-profile > gpurun_out/ncu_update_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_price -s 40 -c 1 -o gpurun_out/prof_price_$TAG python bench.py --steps 60 --warmup 20 --no-cpu-baseline --e2e-max-iter 5 --no-profile > gpurun_out/ncu_price_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pivot -s 40 -c 1 -o gpurun_out/prof_pivot_$TAG python bench.py --steps 60 --warmup 20 --no-cpu-baseline --e2e-max-iter 5 --no-profile > gpurun_out/ncu_pivot_$TAG.log 2>&1
ls gpurun_out
