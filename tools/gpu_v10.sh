# 1 GPU: bench default line with actor stall; event-fix tests; ncu --set full of the pack (launch 2 of 3)
mkdir -p gpurun_out/v10
timeout 300 python bench.py > gpurun_out/v10/bench_n1.log 2>&1
timeout 400 python -m pytest -m gpu -x -q tests/test_gpu_stream_pull.py tests/test_gpu_stress.py > gpurun_out/v10/pytest.log 2>&1; echo rc=$? >> gpurun_out/v10/pytest.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 1 -c 1 -o gpurun_out/v10/pack_sub_full python bench.py --quick --steps 2 --warmup 1 > gpurun_out/v10/ncu_pack.log 2>&1
