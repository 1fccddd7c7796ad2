# 4 GPUs: full GPU test-suite, chain scaling lines N=2/3/4, hop-CTA check, 32B placements (configs 3/4 scaled)
mkdir -p gpurun_out/v9
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/v9/pytest.log 2>&1; echo rc=$? >> gpurun_out/v9/pytest.log
A="--no-e2e --steps 10 --warmup 3"
timeout 200 $TR --nproc-per-node 2 --master-port 29901 bench.py --gpus 2 $A > gpurun_out/v9/chain2.log 2>&1
timeout 200 $TR --nproc-per-node 3 --master-port 29902 bench.py --gpus 3 $A > gpurun_out/v9/chain3.log 2>&1
timeout 200 $TR --nproc-per-node 4 --master-port 29903 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/v9/chain4.log 2>&1
timeout 200 $TR --nproc-per-node 4 --master-port 29904 bench.py --gpus 4 $A --hop-ctas 48 > gpurun_out/v9/chain4_h48.log 2>&1
timeout 200 $TR --nproc-per-node 4 --master-port 29905 bench.py --gpus 4 $A --config colocated --model 32b --tp 4 > gpurun_out/v9/coloc4_32b_tp4.log 2>&1
timeout 200 $TR --nproc-per-node 4 --master-port 29906 bench.py --gpus 4 $A --config colocated --model 32b --tp 2 > gpurun_out/v9/coloc4_32b_tp2.log 2>&1
timeout 200 $TR --nproc-per-node 4 --master-port 29907 bench.py --gpus 4 $A --config relay-tp --model 32b --tp 2 > gpurun_out/v9/relaytp4_32b.log 2>&1
timeout 200 $TR --nproc-per-node 4 --master-port 29908 bench.py --gpus 4 $A --config host > gpurun_out/v9/host4.log 2>&1
