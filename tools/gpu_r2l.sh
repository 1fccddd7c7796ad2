# round 2 (session 3): validate HEAD+lean cast+replica hook on 4 GPUs; CE (host-gated, 2 copy streams) vs kernel; stress
mkdir -p gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2l/smoke.log
LAM_DEBUG_FAIL=1 timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r2l/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2l/pytest4.log
for n in 2 4; do for m in ce kernel; do
timeout 400 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2l/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2l/n${n}_$m.log
done; done
timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2l/stress4.log 2>&1; echo rc=$? >> gpurun_out/r2l/stress4.log
