# 1 GPU: launch list + ncu --set full of the dynamic-distribution pack (N=1 bench command)
mkdir -p gpurun_out/ncu2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu2/launches_n1.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu2/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 1 -c 1 -o gpurun_out/ncu2/pack_sub_full python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu2/ncu_pack.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 1 -c 1 -o gpurun_out/ncu2/pack_plain_full python bench.py --quick --steps 2 --warmup 1 --no-subscribe --stream-pull off > gpurun_out/ncu2/ncu_pack_plain.log 2>&1
