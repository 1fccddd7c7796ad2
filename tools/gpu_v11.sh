# 1 GPU: pack CTA count vs actor-step inflation; host tier with copy-engine hops
mkdir -p gpurun_out/v11
for n in 148 296; do
  timeout 240 python bench.py --no-e2e --no-cpu-baseline --pack-ctas $n > gpurun_out/v11/bench_pack$n.log 2>&1
done
timeout 300 python bench.py --config host --hop-mode ce --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v11/host_ce.log 2>&1
