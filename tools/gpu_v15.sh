# 2 GPUs: multi-GPU parity with the dynamic pull (single- and multi-process), chain N=2 line
mkdir -p gpurun_out/v15
timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_stream_pull.py "tests/test_gpu_multiproc.py::test_multiproc_parity[1]" "tests/test_gpu_multiproc.py::test_multiproc_parity[13]" > gpurun_out/v15/pytest.log 2>&1; echo rc=$? >> gpurun_out/v15/pytest.log
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 2 --no-e2e --steps 10 --warmup 3 > gpurun_out/v15/chain2.log 2>&1
