# ncu launch list of C4 lookaheads (bounded selection) and a full capture of the probe kernels
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_probe.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-max-iter 1 --no-profile --no-reinversion > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_la_probe -s 6 -c 2 -o gpurun_out/prof_probe python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-max-iter 1 --no-profile --no-reinversion > gpurun_out/ncu_probe.log 2>&1
