bash tools/gpu_host4.sh
bash tools/gpu_sweep4.sh
