# 4-GPU chain sweep: hop CTAs x chunk size, streaming pulls on/off (7B, bench default placement)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
A="--gpus 4 --no-e2e --steps 6 --warmup 3"
i=0
for opt in "--hop-ctas 32" "--hop-ctas 64" "--hop-ctas 96" "--hop-ctas 148" "--chunk-mb 64" "--chunk-mb 128" "--hop-ctas 64 --chunk-mb 128" "--stream-pull off" ; do
  i=$((i+1))
  echo "== $opt" >> gpurun_out/v5_sweep.log
  timeout 240 $TR --master-port $((29600+i)) bench.py $A $opt 2>&1 | grep '^{' >> gpurun_out/v5_sweep.log
done
LAM_HOP_PROF=1 timeout 240 $TR --master-port 29690 bench.py $A > gpurun_out/v5_hopprof.log 2>&1
