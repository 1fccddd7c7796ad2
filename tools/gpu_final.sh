# 1 GPU: what the driver runs at round end — smoke, pytest -m gpu, the default bench line
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc=$? >> gpurun_out/final/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest.log 2>&1; echo rc=$? >> gpurun_out/final/pytest.log
timeout 300 python bench.py > gpurun_out/final/bench_n1.log 2>&1
