# round 2 (session 3): hybrid broadcast (multicast share + TMA chain): parity single/multi-process, bench sweep
mkdir -p gpurun_out/r2m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m/build.log 2>&1
export LAM_DEBUG_FAIL=1
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "hybrid or multicast" > gpurun_out/r2m/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest_sp.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -rs -k "17 or 18 or 19 or 21 or 22 or 23" > gpurun_out/r2m/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest_mp.log
for n in 4 2; do for pct in 60 40 75; do
timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode hybrid --mc-pct $pct > gpurun_out/r2m/n${n}_hyb$pct.log 2>&1; echo rc=$? >> gpurun_out/r2m/n${n}_hyb$pct.log
done; done
