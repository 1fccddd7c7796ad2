set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2_pytest4.log 2>&1; echo pytest_rc=$? >> gpurun_out/v2_pytest4.log
timeout 300 $TR --master-port 29511 bench.py --gpus 4 --no-e2e > gpurun_out/v2_chain4.log 2>&1
timeout 300 $TR --master-port 29512 bench.py --gpus 4 --no-e2e --hop-mode ce > gpurun_out/v2_chain4_ce.log 2>&1
timeout 300 $TR --master-port 29513 bench.py --gpus 4 --no-e2e --config colocated --model 32b --tp 4 > gpurun_out/v2_coloc4_32b.log 2>&1
timeout 300 $TR --master-port 29514 bench.py --gpus 4 --no-e2e --config relay-tp --model 32b --tp 2 > gpurun_out/v2_relaytp4_32b.log 2>&1
timeout 300 $TR --master-port 29515 bench.py --gpus 2 --no-e2e > gpurun_out/v2_chain2.log 2>&1
