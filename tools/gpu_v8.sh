# 1 GPU: bench default line (e2e + cpu baseline), host tier, pull microbench, ncu launch list + full captures
mkdir -p gpurun_out/v8
timeout 300 python bench.py > gpurun_out/v8/bench_n1.log 2>&1
timeout 300 python bench.py --config host --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v8/host_n1.log 2>&1
timeout 300 python tools/pull_bench.py --tps 1,2,4 > gpurun_out/v8/pull_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v8/launches_n1.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/v8/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 3 -c 1 -o gpurun_out/v8/pack_full python bench.py --quick --steps 2 --warmup 1 > gpurun_out/v8/ncu_pack.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pull" -s 2 -c 2 -o gpurun_out/v8/pull_full python tools/pull_bench.py --tps 2 --reps 2 > gpurun_out/v8/ncu_pull.log 2>&1
