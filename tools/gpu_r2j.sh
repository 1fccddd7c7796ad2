# round 2 (session 3): CE chain gated on host-mapped ready words; lean cast (cvt.rn.bf16x2 + NaN patch) in k_pack
mkdir -p gpurun_out/r2j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j/build.log 2>&1
timeout 120 ./tools/cvt_probe > gpurun_out/r2j/cvt_probe.log 2>&1
export LAM_DEBUG_FAIL=1
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -rs -k "fullsize or bit_pattern or multicast or chain or corrupt or host or single_gpu or confined" > gpurun_out/r2j/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/r2j/pytest_quick.log
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode ce > gpurun_out/r2j/n2_ce.log 2>&1; echo rc=$? >> gpurun_out/r2j/n2_ce.log
timeout 300 python tools/hop_profile.py 7b 1 --ce > gpurun_out/r2j/hop_sp_ce.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2j/n1.log 2>&1; echo rc=$? >> gpurun_out/r2j/n1.log
