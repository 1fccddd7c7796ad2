# NEXT-3 host-memory relay tier on the box: parity tests, bench placements, pull microbench
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
free -g > gpurun_out/v5_free.txt; nproc >> gpurun_out/v5_free.txt; ulimit -l >> gpurun_out/v5_free.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "host" > gpurun_out/v5_pytest_host.log 2>&1; echo rc=$? >> gpurun_out/v5_pytest_host.log
timeout 300 python bench.py --config host --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v5_host1.log 2>&1
timeout 300 $TR --master-port 29701 bench.py --gpus 4 --config host --no-e2e --steps 3 --warmup 3 > gpurun_out/v5_host4.log 2>&1
timeout 300 python tools/pull_bench.py --tps 1,2,4,8 > gpurun_out/v5_pull_bench.log 2>&1
