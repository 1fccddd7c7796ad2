mkdir -p gpurun_out/r2a
nvidia-smi -L > gpurun_out/r2a/smi.txt; nproc >> gpurun_out/r2a/smi.txt; lscpu | grep "Model name" >> gpurun_out/r2a/smi.txt; free -g >> gpurun_out/r2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2a/pytest4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --no-e2e --steps 10 --warmup 3 > gpurun_out/r2a/chain4.log 2>&1
