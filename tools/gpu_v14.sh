# 1 GPU: dynamic-distribution pull — smoke, pytest -m gpu, pull microbench, bench line; ncu of the new pack
mkdir -p gpurun_out/v14
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v14/smoke.log 2>&1; echo rc=$? >> gpurun_out/v14/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v14/pytest.log 2>&1; echo rc=$? >> gpurun_out/v14/pytest.log
timeout 300 python tools/pull_bench.py --tps 1,2,4 > gpurun_out/v14/pull_bench.log 2>&1
timeout 300 python bench.py > gpurun_out/v14/bench_n1.log 2>&1
bash tools/gpu_ncu2.sh
