# 1 GPU: pack with per-chunk (not per-unit) checksum reduction — parity + bench
mkdir -p gpurun_out/v12
timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_stream_pull.py > gpurun_out/v12/pytest.log 2>&1; echo rc=$? >> gpurun_out/v12/pytest.log
timeout 240 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/v12/bench_n1.log 2>&1
timeout 240 python bench.py --no-e2e --no-cpu-baseline --no-subscribe > gpurun_out/v12/bench_n1_nosub.log 2>&1
