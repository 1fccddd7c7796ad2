# 4 GPUs: k_hop stage geometry 7 x 32 KiB (default) vs 14 x 16 KiB (LAM_HOP_STAGE_KB=16)
mkdir -p gpurun_out/v13
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
A="--no-e2e --no-cpu-baseline --steps 10 --warmup 3"
p=29950
for kb in 32 16; do
  p=$((p+1)); LAM_HOP_STAGE_KB=$kb timeout 200 $TR --nproc-per-node 4 --master-port $p bench.py --gpus 4 $A > gpurun_out/v13/chain4_$kb.log 2>&1
  p=$((p+1)); LAM_HOP_STAGE_KB=$kb timeout 200 $TR --nproc-per-node 2 --master-port $p bench.py --gpus 2 $A > gpurun_out/v13/chain2_$kb.log 2>&1
done
