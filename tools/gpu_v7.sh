# k_hop v5 (flusher warp, 7 stages): parity + repair + selected multi-process tests, chain benches
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_repair.py tests/test_gpu_stream_pull.py "tests/test_gpu_multiproc.py::test_multiproc_parity[3]" "tests/test_gpu_multiproc.py::test_multiproc_parity[7]" "tests/test_gpu_multiproc.py::test_multiproc_parity[6]" > gpurun_out/v7_pytest.log 2>&1; echo rc=$? >> gpurun_out/v7_pytest.log
A="--no-e2e --steps 6 --warmup 3"
timeout 240 $TR --nproc-per-node 4 --master-port 29811 bench.py --gpus 4 $A > gpurun_out/v7_chain4.log 2>&1
LAM_HOP_PROF=1 timeout 240 $TR --nproc-per-node 4 --master-port 29812 bench.py --gpus 4 $A > gpurun_out/v7_chain4_prof.log 2>&1
timeout 240 $TR --nproc-per-node 2 --master-port 29813 bench.py --gpus 2 $A > gpurun_out/v7_chain2.log 2>&1
timeout 240 $TR --nproc-per-node 4 --master-port 29814 bench.py --gpus 4 $A --chunk-mb 128 > gpurun_out/v7_chain4_c128.log 2>&1
