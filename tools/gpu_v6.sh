# k_hop v4 (warp-specialised): parity + repair + multi-process tests, chain bench N=4 / N=2, hop profile
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v6_pytest.log 2>&1; echo rc=$? >> gpurun_out/v6_pytest.log
A="--no-e2e --steps 6 --warmup 3"
timeout 240 $TR --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 $A > gpurun_out/v6_chain4.log 2>&1
LAM_HOP_PROF=1 timeout 240 $TR --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 $A > gpurun_out/v6_chain4_prof.log 2>&1
timeout 240 $TR --nproc-per-node 2 --master-port 29803 bench.py --gpus 2 $A > gpurun_out/v6_chain2.log 2>&1
timeout 240 $TR --nproc-per-node 2 --master-port 29804 bench.py --gpus 2 $A --hop-mode ce > gpurun_out/v6_chain2_ce.log 2>&1
timeout 240 $TR --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 $A --hop-ctas 48 > gpurun_out/v6_chain4_48.log 2>&1
timeout 240 python bench.py --config host $A --no-cpu-baseline --hop-ctas 148 > gpurun_out/v6_host1_148.log 2>&1
