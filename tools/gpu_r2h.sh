# round 2 (session 3): device-gated copy-engine chain + k_hop pred-verdict check: full GPU suite, CE vs kernel bench, pack per-SM bench
mkdir -p gpurun_out/r2h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h/build.log 2>&1
timeout 200 ./tools/pack_sm_bench > gpurun_out/r2h/pack_sm_bench.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "chain or host or corrupt or multicast" > gpurun_out/r2h/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/r2h/pytest_quick.log
for n in 2 4; do for m in ce kernel; do
timeout 400 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2h/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2h/n${n}_$m.log
done; done
timeout 1800 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2h/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/r2h/pytest_all.log
