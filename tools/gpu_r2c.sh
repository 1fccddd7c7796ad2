# round 2: host-gated copy-engine hops vs k_hop; stress reordered; NVLink counters; full-size parity tests
mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c/build.log 2>&1
nvidia-smi nvlink -gt d -i 1 > gpurun_out/r2c/nvlink_gt_before.txt 2>&1
nvidia-smi nvlink -s -i 1 > gpurun_out/r2c/nvlink_status.txt 2>&1
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --hop-mode ce > gpurun_out/r2c/n4_ce.log 2>&1
nvidia-smi nvlink -gt d -i 1 > gpurun_out/r2c/nvlink_gt_after.txt 2>&1
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r2c/n4_kernel.log 2>&1
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --hop-mode ce > gpurun_out/r2c/n2_ce.log 2>&1
timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2c/stress4.log 2>&1
timeout 600 python bench.py --config stress --stress-steps 40 > gpurun_out/r2c/stress1.log 2>&1
timeout 300 python tools/hop_profile.py > gpurun_out/r2c/hop_profile.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_hop --csv --log-file gpurun_out/r2c/hop_ncu.csv python tools/hop_profile.py > gpurun_out/r2c/hop_ncu.log 2>&1
timeout 1200 python -m pytest -q -x tests/test_gpu_fullsize.py "tests/test_gpu_parity.py::test_7b_single_gpu_all_headers_sampled_elements" "tests/test_gpu_parity.py::test_corrupt_chunk_is_never_committed" "tests/test_gpu_parity.py::test_tiny_chain_across_gpus" "tests/test_gpu_parity.py::test_tiny_three_versions_chain_on_one_gpu" > gpurun_out/r2c/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/r2c/pytest_new.log
timeout 900 python -m pytest -q -x tests/test_gpu_multiproc.py tests/test_gpu_repair.py > gpurun_out/r2c/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2c/pytest_mp.log
