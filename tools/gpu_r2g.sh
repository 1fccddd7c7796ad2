# round 2 (session 3): NEXT-2 multicast hop mode — parity (single- and multi-process), bench mc vs kernel vs CE
mkdir -p gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g/build.log 2>&1
timeout 120 ./tools/mc_bench > gpurun_out/r2g/mc_bench.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "multicast" -rs > gpurun_out/r2g/pytest_mc.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest_mc.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -rs -k "17 or 18 or 19" > gpurun_out/r2g/pytest_mc_mp.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest_mc_mp.log
for n in 2 4; do for m in mc ce; do
timeout 400 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2g/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2g/n${n}_$m.log
done; done
