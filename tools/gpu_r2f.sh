# round 2 (session 3): chain transport choice — chain_bench (pull/push TMA, reg, split, CE), IPC CE,
# single-process hop timings (kernel vs CE), NVLink counters of k_hop (ncu), nvidia-smi link counters
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f/build.log 2>&1
timeout 300 ./tools/chain_bench > gpurun_out/r2f/chain_bench.log 2>&1
timeout 300 python tools/ipc_ce_bench.py > gpurun_out/r2f/ipc_ce.log 2>&1
for m in "" "--ce"; do for k in 1 3; do timeout 300 python tools/hop_profile.py 7b $k $m >> gpurun_out/r2f/hop_sp.log 2>&1; done; done
timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes.sum.per_second,nvltx__bytes.sum.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_hop --csv --log-file gpurun_out/r2f/hop_ncu.csv python tools/hop_profile.py 7b 1 > gpurun_out/r2f/hop_ncu.log 2>&1
for d in 0 1 2 3; do nvidia-smi nvlink -gt d -i $d > gpurun_out/r2f/nvl_before_$d.txt 2>&1; done
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 3 --quick --no-verify > gpurun_out/r2f/n4_quick.log 2>&1
for d in 0 1 2 3; do nvidia-smi nvlink -gt d -i $d > gpurun_out/r2f/nvl_after_$d.txt 2>&1; done
