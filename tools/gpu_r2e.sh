# round 2 (session 3): validate HEAD on 4 GPUs — smoke, full pytest -m gpu, bench N=1/2/4, stress
mkdir -p gpurun_out/r2e
(nvidia-smi -L; nproc; lscpu | grep "Model name"; free -g) > gpurun_out/r2e/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2e/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x -rs --durations=15 > gpurun_out/r2e/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2e/pytest4.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2e/n1.log 2>&1; echo rc=$? >> gpurun_out/r2e/n1.log
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2e/n2.log 2>&1; echo rc=$? >> gpurun_out/r2e/n2.log
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2e/n4.log 2>&1; echo rc=$? >> gpurun_out/r2e/n4.log
timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2e/stress4.log 2>&1; echo rc=$? >> gpurun_out/r2e/stress4.log
