# round 2 (session 3): profiles — bench N=1 (driver's K/W), launch list, ncu full capture of the pack,
# NVLink counters of the multicast pack (single-process 2 GPUs), smoke
mkdir -p gpurun_out/r2n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2n/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n/n1.log 2>&1; echo rc=$? >> gpurun_out/r2n/n1.log
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n/launches_n1.csv python bench.py --steps 2 --warmup 1 --quick --no-verify > gpurun_out/r2n/ncu_launch.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pack -s 2 -c 1 -o gpurun_out/r2n/pack_subscriber_full python bench.py --steps 2 --warmup 1 --quick --no-verify > gpurun_out/r2n/ncu_full.log 2>&1
timeout 300 python tools/mc_profile.py > gpurun_out/r2n/mc_profile.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes.sum.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pack --csv --log-file gpurun_out/r2n/mc_pack_ncu.csv python tools/mc_profile.py > gpurun_out/r2n/mc_ncu.log 2>&1
