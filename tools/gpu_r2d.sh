# round 2: why copy-engine hops are slow in the multi-process runtime (IPC vs peer), single-process chains
mkdir -p gpurun_out/r2d
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d/build.log 2>&1
timeout 300 python tools/ipc_ce_bench.py > gpurun_out/r2d/ipc_ce.log 2>&1
for m in "" "--ce"; do for k in 1 3; do timeout 300 python tools/hop_profile.py 7b $k $m >> gpurun_out/r2d/hop_sp.log 2>&1; done; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2d/n1_stall.log 2>&1
timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 --stress-ms 50 > gpurun_out/r2d/stress4_50.log 2>&1
timeout 600 python bench.py --config stress --stress-steps 40 --slots 3 > gpurun_out/r2d/stress1_s3.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_repair.py tests/test_gpu_parity.py -k "confined or sigkill" > gpurun_out/r2d/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2d/pytest.log
