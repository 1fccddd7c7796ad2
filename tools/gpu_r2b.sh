# round 2: transport microbenchmark + new bench (N=1 full line, N=4 self-launch, stress, headline at N=4, reference arm)
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
timeout 300 ./tools/chain_bench > gpurun_out/r2b/chain_bench.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b/n1.log 2>&1
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r2b/n4.log 2>&1
timeout 600 python bench.py --gpus 4 --config stress --stress-steps 30 > gpurun_out/r2b/stress4.log 2>&1
timeout 900 python bench.py --gpus 4 --steps 3 --warmup 1 --no-e2e --headline on --extra-steps 3 > gpurun_out/r2b/headline4.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b/ref1.log 2>&1
