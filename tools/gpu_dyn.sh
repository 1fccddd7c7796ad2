# 1 GPU: what the driver runs at round end — smoke, pytest -m gpu, the default bench line
mkdir -p gpurun_out/dyn
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dyn/smoke.log 2>&1; echo rc=$? >> gpurun_out/dyn/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dyn/pytest.log 2>&1; echo rc=$? >> gpurun_out/dyn/pytest.log
timeout 300 python bench.py > gpurun_out/dyn/bench_n1.log 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-subscribe --stream-pull off > gpurun_out/dyn/bench_n1_nosub.log 2>&1
