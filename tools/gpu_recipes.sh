#!/bin/bash
# Every gpurun recipe used to produce profiles/ (round 1: v5..v15, n4, sweep4, host4, ncu2, dyn, final;
# round 2: r2a..r2n), one shell function each, run from the repo root on the GPU box:
#   /usr/local/graft/bin/gpurun --gpus 4 --timeout 3000 -- "bash tools/gpu_recipes.sh r2l"
# Outputs land in gpurun_out/<recipe>/ (scratch); the ones worth keeping are copied to profiles/.
set -u

recipe_sweep4() {
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
}

recipe_n4() {
  set -x
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2_pytest4.log 2>&1; echo pytest_rc=$? >> gpurun_out/v2_pytest4.log
  timeout 300 $TR --master-port 29511 bench.py --gpus 4 --no-e2e > gpurun_out/v2_chain4.log 2>&1
  timeout 300 $TR --master-port 29512 bench.py --gpus 4 --no-e2e --hop-mode ce > gpurun_out/v2_chain4_ce.log 2>&1
  timeout 300 $TR --master-port 29513 bench.py --gpus 4 --no-e2e --config colocated --model 32b --tp 4 > gpurun_out/v2_coloc4_32b.log 2>&1
  timeout 300 $TR --master-port 29514 bench.py --gpus 4 --no-e2e --config relay-tp --model 32b --tp 2 > gpurun_out/v2_relaytp4_32b.log 2>&1
  timeout 300 $TR --master-port 29515 bench.py --gpus 2 --no-e2e > gpurun_out/v2_chain2.log 2>&1
}

recipe_v9() {
  # 4 GPUs: full GPU test-suite, chain scaling lines N=2/3/4, hop-CTA check, 32B placements (configs 3/4 scaled)
  mkdir -p gpurun_out/v9
  TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
  timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/v9/pytest.log 2>&1; echo rc=$? >> gpurun_out/v9/pytest.log
  A="--no-e2e --steps 10 --warmup 3"
  timeout 200 $TR --nproc-per-node 2 --master-port 29901 bench.py --gpus 2 $A > gpurun_out/v9/chain2.log 2>&1
  timeout 200 $TR --nproc-per-node 3 --master-port 29902 bench.py --gpus 3 $A > gpurun_out/v9/chain3.log 2>&1
  timeout 200 $TR --nproc-per-node 4 --master-port 29903 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/v9/chain4.log 2>&1
  timeout 200 $TR --nproc-per-node 4 --master-port 29904 bench.py --gpus 4 $A --hop-ctas 48 > gpurun_out/v9/chain4_h48.log 2>&1
  timeout 200 $TR --nproc-per-node 4 --master-port 29905 bench.py --gpus 4 $A --config colocated --model 32b --tp 4 > gpurun_out/v9/coloc4_32b_tp4.log 2>&1
  timeout 200 $TR --nproc-per-node 4 --master-port 29906 bench.py --gpus 4 $A --config colocated --model 32b --tp 2 > gpurun_out/v9/coloc4_32b_tp2.log 2>&1
  timeout 200 $TR --nproc-per-node 4 --master-port 29907 bench.py --gpus 4 $A --config relay-tp --model 32b --tp 2 > gpurun_out/v9/relaytp4_32b.log 2>&1
  timeout 200 $TR --nproc-per-node 4 --master-port 29908 bench.py --gpus 4 $A --config host > gpurun_out/v9/host4.log 2>&1
}

recipe_v10() {
  # 1 GPU: bench default line with actor stall; event-fix tests; ncu --set full of the pack (launch 2 of 3)
  mkdir -p gpurun_out/v10
  timeout 300 python bench.py > gpurun_out/v10/bench_n1.log 2>&1
  timeout 400 python -m pytest -m gpu -x -q tests/test_gpu_stream_pull.py tests/test_gpu_stress.py > gpurun_out/v10/pytest.log 2>&1; echo rc=$? >> gpurun_out/v10/pytest.log
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 1 -c 1 -o gpurun_out/v10/pack_sub_full python bench.py --quick --steps 2 --warmup 1 > gpurun_out/v10/ncu_pack.log 2>&1
}

recipe_v15() {
  # 2 GPUs: multi-GPU parity with the dynamic pull (single- and multi-process), chain N=2 line
  mkdir -p gpurun_out/v15
  timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_stream_pull.py "tests/test_gpu_multiproc.py::test_multiproc_parity[1]" "tests/test_gpu_multiproc.py::test_multiproc_parity[13]" > gpurun_out/v15/pytest.log 2>&1; echo rc=$? >> gpurun_out/v15/pytest.log
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 2 --no-e2e --steps 10 --warmup 3 > gpurun_out/v15/chain2.log 2>&1
}

recipe_host4() {
  # NEXT-3 host-memory relay tier on the box: parity tests, bench placements, pull microbench
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
  free -g > gpurun_out/v5_free.txt; nproc >> gpurun_out/v5_free.txt; ulimit -l >> gpurun_out/v5_free.txt
  timeout 900 python -m pytest tests -m gpu -x -q -k "host" > gpurun_out/v5_pytest_host.log 2>&1; echo rc=$? >> gpurun_out/v5_pytest_host.log
  timeout 300 python bench.py --config host --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v5_host1.log 2>&1
  timeout 300 $TR --master-port 29701 bench.py --gpus 4 --config host --no-e2e --steps 3 --warmup 3 > gpurun_out/v5_host4.log 2>&1
  timeout 300 python tools/pull_bench.py --tps 1,2,4,8 > gpurun_out/v5_pull_bench.log 2>&1
}

recipe_v5() {
  bash tools/gpu_host4.sh
  bash tools/gpu_sweep4.sh
}

recipe_v12() {
  # 1 GPU: pack with per-chunk (not per-unit) checksum reduction — parity + bench
  mkdir -p gpurun_out/v12
  timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_stream_pull.py > gpurun_out/v12/pytest.log 2>&1; echo rc=$? >> gpurun_out/v12/pytest.log
  timeout 240 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/v12/bench_n1.log 2>&1
  timeout 240 python bench.py --no-e2e --no-cpu-baseline --no-subscribe > gpurun_out/v12/bench_n1_nosub.log 2>&1
}

recipe_dyn() {
  # 1 GPU: what the driver runs at round end — smoke, pytest -m gpu, the default bench line
  mkdir -p gpurun_out/dyn
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dyn/smoke.log 2>&1; echo rc=$? >> gpurun_out/dyn/smoke.log
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dyn/pytest.log 2>&1; echo rc=$? >> gpurun_out/dyn/pytest.log
  timeout 300 python bench.py > gpurun_out/dyn/bench_n1.log 2>&1
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-subscribe --stream-pull off > gpurun_out/dyn/bench_n1_nosub.log 2>&1
}

recipe_v13() {
  # 4 GPUs: k_hop stage geometry 7 x 32 KiB (default) vs 14 x 16 KiB (LAM_HOP_STAGE_KB=16)
  mkdir -p gpurun_out/v13
  TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
  A="--no-e2e --no-cpu-baseline --steps 10 --warmup 3"
  p=29950
  for kb in 32 16; do
    p=$((p+1)); LAM_HOP_STAGE_KB=$kb timeout 200 $TR --nproc-per-node 4 --master-port $p bench.py --gpus 4 $A > gpurun_out/v13/chain4_$kb.log 2>&1
    p=$((p+1)); LAM_HOP_STAGE_KB=$kb timeout 200 $TR --nproc-per-node 2 --master-port $p bench.py --gpus 2 $A > gpurun_out/v13/chain2_$kb.log 2>&1
  done
}

recipe_final() {
  # 1 GPU: what the driver runs at round end — smoke, pytest -m gpu, the default bench line
  mkdir -p gpurun_out/final
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc=$? >> gpurun_out/final/smoke.log
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest.log 2>&1; echo rc=$? >> gpurun_out/final/pytest.log
  timeout 300 python bench.py > gpurun_out/final/bench_n1.log 2>&1
}

recipe_r2c() {
  # round 2: host-gated copy-engine hops vs k_hop; stress reordered; NVLink counters; full-size parity tests
  mkdir -p gpurun_out/r2c
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c/build.log 2>&1
  nvidia-smi nvlink -gt d -i 1 > gpurun_out/r2c/nvlink_gt_before.txt 2>&1
  nvidia-smi nvlink -s -i 1 > gpurun_out/r2c/nvlink_status.txt 2>&1
  timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --hop-mode ce > gpurun_out/r2c/n4_ce.log 2>&1
  nvidia-smi nvlink -gt d -i 1 > gpurun_out/r2c/nvlink_gt_after.txt 2>&1
  timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r2c/n4_kernel.log 2>&1
  timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --hop-mode ce > gpurun_out/r2c/n2_ce.log 2>&1
  timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2c/stress4.log 2>&1
  timeout 600 python bench.py --config stress --stress-steps 40 > gpurun_out/r2c/stress1.log 2>&1
  timeout 300 python tools/hop_profile.py > gpurun_out/r2c/hop_profile.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_hop --csv --log-file gpurun_out/r2c/hop_ncu.csv python tools/hop_profile.py > gpurun_out/r2c/hop_ncu.log 2>&1
  timeout 1200 python -m pytest -q -x tests/test_gpu_fullsize.py "tests/test_gpu_parity.py::test_7b_single_gpu_all_headers_sampled_elements" "tests/test_gpu_parity.py::test_corrupt_chunk_is_never_committed" "tests/test_gpu_parity.py::test_tiny_chain_across_gpus" "tests/test_gpu_parity.py::test_tiny_three_versions_chain_on_one_gpu" > gpurun_out/r2c/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/r2c/pytest_new.log
  timeout 900 python -m pytest -q -x tests/test_gpu_multiproc.py tests/test_gpu_repair.py > gpurun_out/r2c/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2c/pytest_mp.log
}

recipe_v14() {
  # 1 GPU: dynamic-distribution pull — smoke, pytest -m gpu, pull microbench, bench line; ncu of the new pack
  mkdir -p gpurun_out/v14
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v14/smoke.log 2>&1; echo rc=$? >> gpurun_out/v14/smoke.log
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v14/pytest.log 2>&1; echo rc=$? >> gpurun_out/v14/pytest.log
  timeout 300 python tools/pull_bench.py --tps 1,2,4 > gpurun_out/v14/pull_bench.log 2>&1
  timeout 300 python bench.py > gpurun_out/v14/bench_n1.log 2>&1
  bash tools/gpu_ncu2.sh
}

recipe_r2b() {
  # round 2: transport microbenchmark + new bench (N=1 full line, N=4 self-launch, stress, headline at N=4, reference arm)
  mkdir -p gpurun_out/r2b
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
  timeout 300 ./tools/chain_bench > gpurun_out/r2b/chain_bench.log 2>&1
  timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b/n1.log 2>&1
  timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r2b/n4.log 2>&1
  timeout 600 python bench.py --gpus 4 --config stress --stress-steps 30 > gpurun_out/r2b/stress4.log 2>&1
  timeout 900 python bench.py --gpus 4 --steps 3 --warmup 1 --no-e2e --headline on --extra-steps 3 > gpurun_out/r2b/headline4.log 2>&1
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b/ref1.log 2>&1
}

recipe_ncu2() {
  # 1 GPU: launch list + ncu --set full of the dynamic-distribution pack (N=1 bench command)
  mkdir -p gpurun_out/ncu2
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu2/launches_n1.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu2/ncu_launch.log 2>&1
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 1 -c 1 -o gpurun_out/ncu2/pack_sub_full python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu2/ncu_pack.log 2>&1
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 1 -c 1 -o gpurun_out/ncu2/pack_plain_full python bench.py --quick --steps 2 --warmup 1 --no-subscribe --stream-pull off > gpurun_out/ncu2/ncu_pack_plain.log 2>&1
}

recipe_v7() {
  # k_hop v5 (flusher warp, 7 stages): parity + repair + selected multi-process tests, chain benches
  TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
  timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_repair.py tests/test_gpu_stream_pull.py "tests/test_gpu_multiproc.py::test_multiproc_parity[3]" "tests/test_gpu_multiproc.py::test_multiproc_parity[7]" "tests/test_gpu_multiproc.py::test_multiproc_parity[6]" > gpurun_out/v7_pytest.log 2>&1; echo rc=$? >> gpurun_out/v7_pytest.log
  A="--no-e2e --steps 6 --warmup 3"
  timeout 240 $TR --nproc-per-node 4 --master-port 29811 bench.py --gpus 4 $A > gpurun_out/v7_chain4.log 2>&1
  LAM_HOP_PROF=1 timeout 240 $TR --nproc-per-node 4 --master-port 29812 bench.py --gpus 4 $A > gpurun_out/v7_chain4_prof.log 2>&1
  timeout 240 $TR --nproc-per-node 2 --master-port 29813 bench.py --gpus 2 $A > gpurun_out/v7_chain2.log 2>&1
  timeout 240 $TR --nproc-per-node 4 --master-port 29814 bench.py --gpus 4 $A --chunk-mb 128 > gpurun_out/v7_chain4_c128.log 2>&1
}

recipe_r2d() {
  # round 2: why copy-engine hops are slow in the multi-process runtime (IPC vs peer), single-process chains
  mkdir -p gpurun_out/r2d
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d/build.log 2>&1
  timeout 300 python tools/ipc_ce_bench.py > gpurun_out/r2d/ipc_ce.log 2>&1
  for m in "" "--ce"; do for k in 1 3; do timeout 300 python tools/hop_profile.py 7b $k $m >> gpurun_out/r2d/hop_sp.log 2>&1; done; done
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2d/n1_stall.log 2>&1
  timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 --stress-ms 50 > gpurun_out/r2d/stress4_50.log 2>&1
  timeout 600 python bench.py --config stress --stress-steps 40 --slots 3 > gpurun_out/r2d/stress1_s3.log 2>&1
  timeout 900 python -m pytest -q -x tests/test_gpu_repair.py tests/test_gpu_parity.py -k "confined or sigkill" > gpurun_out/r2d/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2d/pytest.log
}

recipe_r2a() {
  mkdir -p gpurun_out/r2a
  nvidia-smi -L > gpurun_out/r2a/smi.txt; nproc >> gpurun_out/r2a/smi.txt; lscpu | grep "Model name" >> gpurun_out/r2a/smi.txt; free -g >> gpurun_out/r2a/smi.txt
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2a/pytest4.log
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --no-e2e --steps 10 --warmup 3 > gpurun_out/r2a/chain4.log 2>&1
}

recipe_v11() {
  # 1 GPU: pack CTA count vs actor-step inflation; host tier with copy-engine hops
  mkdir -p gpurun_out/v11
  for n in 148 296; do
    timeout 240 python bench.py --no-e2e --no-cpu-baseline --pack-ctas $n > gpurun_out/v11/bench_pack$n.log 2>&1
  done
  timeout 300 python bench.py --config host --hop-mode ce --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v11/host_ce.log 2>&1
}

recipe_v6() {
  # k_hop v4 (warp-specialised): parity + repair + multi-process tests, chain bench N=4 / N=2, hop profile
  TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v6_pytest.log 2>&1; echo rc=$? >> gpurun_out/v6_pytest.log
  A="--no-e2e --steps 6 --warmup 3"
  timeout 240 $TR --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 $A > gpurun_out/v6_chain4.log 2>&1
  LAM_HOP_PROF=1 timeout 240 $TR --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 $A > gpurun_out/v6_chain4_prof.log 2>&1
  timeout 240 $TR --nproc-per-node 2 --master-port 29803 bench.py --gpus 2 $A > gpurun_out/v6_chain2.log 2>&1
  timeout 240 $TR --nproc-per-node 2 --master-port 29804 bench.py --gpus 2 $A --hop-mode ce > gpurun_out/v6_chain2_ce.log 2>&1
  timeout 240 $TR --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 $A --hop-ctas 48 > gpurun_out/v6_chain4_48.log 2>&1
  timeout 240 python bench.py --config host $A --no-cpu-baseline --hop-ctas 148 > gpurun_out/v6_host1_148.log 2>&1
}

recipe_v8() {
  # 1 GPU: bench default line (e2e + cpu baseline), host tier, pull microbench, ncu launch list + full captures
  mkdir -p gpurun_out/v8
  timeout 300 python bench.py > gpurun_out/v8/bench_n1.log 2>&1
  timeout 300 python bench.py --config host --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v8/host_n1.log 2>&1
  timeout 300 python tools/pull_bench.py --tps 1,2,4 > gpurun_out/v8/pull_bench.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v8/launches_n1.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/v8/ncu_launch.log 2>&1
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pack" -s 3 -c 1 -o gpurun_out/v8/pack_full python bench.py --quick --steps 2 --warmup 1 > gpurun_out/v8/ncu_pack.log 2>&1
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_pull" -s 2 -c 2 -o gpurun_out/v8/pull_full python tools/pull_bench.py --tps 2 --reps 2 > gpurun_out/v8/ncu_pull.log 2>&1
}

recipe_r2e() {
  # round 2 (session 3): validate HEAD on 4 GPUs — smoke, full pytest -m gpu, bench N=1/2/4, stress
  mkdir -p gpurun_out/r2e
  (nvidia-smi -L; nproc; lscpu | grep "Model name"; free -g) > gpurun_out/r2e/box.txt 2>&1
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2e/smoke.log
  timeout 1800 python -m pytest tests -m gpu -q -x -rs --durations=15 > gpurun_out/r2e/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2e/pytest4.log
  timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2e/n1.log 2>&1; echo rc=$? >> gpurun_out/r2e/n1.log
  timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2e/n2.log 2>&1; echo rc=$? >> gpurun_out/r2e/n2.log
  timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2e/n4.log 2>&1; echo rc=$? >> gpurun_out/r2e/n4.log
  timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2e/stress4.log 2>&1; echo rc=$? >> gpurun_out/r2e/stress4.log
}

recipe_r2f() {
  # round 2 (session 3): chain transport choice — chain_bench (pull/push TMA, reg, split, CE), IPC CE,
  # single-process hop timings (kernel vs CE), NVLink counters of k_hop (ncu), nvidia-smi link counters
  mkdir -p gpurun_out/r2f
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f/build.log 2>&1
  timeout 300 ./tools/chain_bench > gpurun_out/r2f/chain_bench.log 2>&1
  timeout 300 python tools/ipc_ce_bench.py > gpurun_out/r2f/ipc_ce.log 2>&1
  for m in "" "--ce"; do for k in 1 3; do timeout 300 python tools/hop_profile.py 7b $k $m >> gpurun_out/r2f/hop_sp.log 2>&1; done; done
  timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes.sum.per_second,nvltx__bytes.sum.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_hop --csv --log-file gpurun_out/r2f/hop_ncu.csv python tools/hop_profile.py 7b 1 > gpurun_out/r2f/hop_ncu.log 2>&1
  for d in 0 1 2 3; do nvidia-smi nvlink -gt d -i $d > gpurun_out/r2f/nvl_before_$d.txt 2>&1; done
  timeout 600 python bench.py --gpus 4 --steps 20 --warmup 3 --quick --no-verify > gpurun_out/r2f/n4_quick.log 2>&1
  for d in 0 1 2 3; do nvidia-smi nvlink -gt d -i $d > gpurun_out/r2f/nvl_after_$d.txt 2>&1; done
}

recipe_r2g() {
  # round 2 (session 3): NEXT-2 multicast hop mode — parity (single- and multi-process), bench mc vs kernel vs CE
  mkdir -p gpurun_out/r2g
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g/build.log 2>&1
  timeout 120 ./tools/mc_bench > gpurun_out/r2g/mc_bench.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "multicast" -rs > gpurun_out/r2g/pytest_mc.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest_mc.log
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -rs -k "17 or 18 or 19" > gpurun_out/r2g/pytest_mc_mp.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest_mc_mp.log
  for n in 2 4; do for m in mc ce; do
  timeout 400 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2g/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2g/n${n}_$m.log
  done; done
}

recipe_r2h() {
  # round 2 (session 3): device-gated copy-engine chain + k_hop pred-verdict check: full GPU suite, CE vs kernel bench, pack per-SM bench
  mkdir -p gpurun_out/r2h
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h/build.log 2>&1
  timeout 200 ./tools/pack_sm_bench > gpurun_out/r2h/pack_sm_bench.log 2>&1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "chain or host or corrupt or multicast" > gpurun_out/r2h/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/r2h/pytest_quick.log
  for n in 2 4; do for m in ce kernel; do
  timeout 400 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2h/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2h/n${n}_$m.log
  done; done
  timeout 1800 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2h/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/r2h/pytest_all.log
}

recipe_r2j() {
  # round 2 (session 3): CE chain gated on host-mapped ready words; lean cast (cvt.rn.bf16x2 + NaN patch) in k_pack
  mkdir -p gpurun_out/r2j
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j/build.log 2>&1
  timeout 120 ./tools/cvt_probe > gpurun_out/r2j/cvt_probe.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -rs -k "fullsize or bit_pattern or multicast or chain or corrupt or host or single_gpu or confined" > gpurun_out/r2j/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/r2j/pytest_quick.log
  timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode ce > gpurun_out/r2j/n2_ce.log 2>&1; echo rc=$? >> gpurun_out/r2j/n2_ce.log
  timeout 300 python tools/hop_profile.py 7b 1 --ce > gpurun_out/r2j/hop_sp_ce.log 2>&1
  timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2j/n1.log 2>&1; echo rc=$? >> gpurun_out/r2j/n1.log
}

recipe_r2l() {
  # round 2 (session 3): validate HEAD+lean cast+replica hook on 4 GPUs; CE (host-gated, 2 copy streams) vs kernel; stress
  mkdir -p gpurun_out/r2l
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2l/smoke.log
  LAM_DEBUG_FAIL=1 timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r2l/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2l/pytest4.log
  for n in 2 4; do for m in ce kernel; do
  timeout 400 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2l/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2l/n${n}_$m.log
  done; done
  timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2l/stress4.log 2>&1; echo rc=$? >> gpurun_out/r2l/stress4.log
}

recipe_r2m() {
  # round 2 (session 3): hybrid broadcast (multicast share + TMA chain): parity single/multi-process, bench sweep
  mkdir -p gpurun_out/r2m
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "hybrid or multicast" > gpurun_out/r2m/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest_sp.log
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -rs -k "17 or 18 or 19 or 21 or 22 or 23" > gpurun_out/r2m/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest_mp.log
  for n in 4 2; do for pct in 60 40 75; do
  timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode hybrid --mc-pct $pct > gpurun_out/r2m/n${n}_hyb$pct.log 2>&1; echo rc=$? >> gpurun_out/r2m/n${n}_hyb$pct.log
  done; done
}

recipe_r2n() {
  # round 2 (session 3): profiles — bench N=1 (driver's K/W), launch list, ncu full capture of the pack,
  # NVLink counters of the multicast pack (single-process 2 GPUs), smoke
  mkdir -p gpurun_out/r2n
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2n/smoke.log
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n/n1.log 2>&1; echo rc=$? >> gpurun_out/r2n/n1.log
  CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n/launches_n1.csv python bench.py --steps 2 --warmup 1 --quick --no-verify > gpurun_out/r2n/ncu_launch.log 2>&1
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pack -s 2 -c 1 -o gpurun_out/r2n/pack_subscriber_full python bench.py --steps 2 --warmup 1 --quick --no-verify > gpurun_out/r2n/ncu_full.log 2>&1
  timeout 300 python tools/mc_profile.py > gpurun_out/r2n/mc_profile.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes.sum.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pack --csv --log-file gpurun_out/r2n/mc_pack_ncu.csv python tools/mc_profile.py > gpurun_out/r2n/mc_ncu.log 2>&1
}

recipe_r2o() {
  # does a slower, SM-confined pack leave GPU 0's HBM to the first hop's peer reads? (chain N=2/4)
  mkdir -p gpurun_out/r2o
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o/build.log 2>&1
  for n in 2 4; do for k in 48 80; do
  timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --pack-sms $k > gpurun_out/r2o/n${n}_sms$k.log 2>&1; echo rc=$? >> gpurun_out/r2o/n${n}_sms$k.log
  done; done
}

recipe_r2p() {
  # does the relay's streaming reshard slow its hop? (chain N=2: pulls streamed with fewer CTAs / not streamed)
  mkdir -p gpurun_out/r2p
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p/build.log 2>&1
  timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --stream-pull off > gpurun_out/r2p/n2_nostream.log 2>&1
  for k in 24 48; do
  timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --pull-ctas $k > gpurun_out/r2p/n2_pull$k.log 2>&1
  done
  timeout 300 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --pull-ctas 48 > gpurun_out/r2p/n4_pull48.log 2>&1
}

recipe_r2q() {
  # host-memory relay tier (NEXT-3): k_hop with TMA bulk stores into pinned host memory vs 16-B stores
  mkdir -p gpurun_out/r2q
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q/build.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "host" > gpurun_out/r2q/pytest_host.log 2>&1; echo rc=$? >> gpurun_out/r2q/pytest_host.log
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -rs -k "14 or 15 or 16" > gpurun_out/r2q/pytest_host_mp.log 2>&1; echo rc=$? >> gpurun_out/r2q/pytest_host_mp.log
  for h in 32 96; do
  timeout 600 python bench.py --config host --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --hop-ctas $h > gpurun_out/r2q/host_n1_bulk_h$h.log 2>&1
  LAM_HOP_NO_BULK=1 timeout 600 python bench.py --config host --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --hop-ctas $h > gpurun_out/r2q/host_n1_st_h$h.log 2>&1
  done
  timeout 600 python bench.py --gpus 2 --config host --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2q/host_n2_bulk.log 2>&1
}

recipe_r2r() {
  # copy-engine chain v3 (progress thread + verify-only k_hop) and k_hop's predecessor-verdict check:
  # full GPU suite on 4 GPUs, CE vs kernel chain
  mkdir -p gpurun_out/r2r
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "chain or host or corrupt" > gpurun_out/r2r/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/r2r/pytest_quick.log
  for n in 2 4; do
  timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode ce > gpurun_out/r2r/n${n}_ce.log 2>&1; echo rc=$? >> gpurun_out/r2r/n${n}_ce.log
  done
  timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/r2r/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2r/pytest4.log
}

recipe_r2s() {
  # copy-engine chain v3 with stream-ordered plan allocations: parity (incl. 7B CE + streaming pulls) and bench
  mkdir -p gpurun_out/r2s
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -rs -k "8 or 9 or 16 or 20 or 21" > gpurun_out/r2s/pytest_mp_ce.log 2>&1; echo rc=$? >> gpurun_out/r2s/pytest_mp_ce.log
  for n in 2 4; do for m in ce kernel; do
  timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode $m > gpurun_out/r2s/n${n}_$m.log 2>&1; echo rc=$? >> gpurun_out/r2s/n${n}_$m.log
  done; done
}

recipe_r2t() {
  # debug: copy-engine chain stall at the first chunk past the enqueue window (bench N=2)
  mkdir -p gpurun_out/r2t
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t/build.log 2>&1
  LAM_DEBUG_FAIL=1 LAM_DEBUG_CE=1 timeout 200 python bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-verify --hop-mode ce > gpurun_out/r2t/n2_ce.log 2>&1
  LAM_DEBUG_FAIL=1 LAM_DEBUG_CE=1 timeout 200 python bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-verify --hop-mode ce --stream-pull off > gpurun_out/r2t/n2_ce_nostream.log 2>&1
}

recipe_r2u() {
  # debug: copy-engine chain stall with streaming pulls — more hardware queues / one copy stream
  mkdir -p gpurun_out/r2u
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u/build.log 2>&1
  export LAM_DEBUG_FAIL=1 LAM_DEBUG_CE=1
  CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 200 python bench.py --gpus 2 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-verify --hop-mode ce > gpurun_out/r2u/n2_ce_conn32.log 2>&1
  LAM_CE_ONE_STREAM=1 timeout 200 python bench.py --gpus 2 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-verify --hop-mode ce > gpurun_out/r2u/n2_ce_one.log 2>&1
}

recipe_r2v() {
  # round-2 final validation on 4 GPUs: smoke, pytest -m gpu, bench N=1 (driver K/W), N=2/4 chain,
  # N=4 multicast, stress, reference arm
  mkdir -p gpurun_out/r2v
  (nvidia-smi -L; nproc; lscpu | grep "Model name") > gpurun_out/r2v/box.txt 2>&1
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2v/smoke.log
  LAM_DEBUG_FAIL=1 timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r2v/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2v/pytest4.log
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2v/n1.log 2>&1; echo rc=$? >> gpurun_out/r2v/n1.log
  for n in 2 4; do
  timeout 400 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2v/n$n.log 2>&1; echo rc=$? >> gpurun_out/r2v/n$n.log
  done
  timeout 400 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode mc > gpurun_out/r2v/n4_mc.log 2>&1; echo rc=$? >> gpurun_out/r2v/n4_mc.log
  timeout 600 python bench.py --gpus 4 --config stress --stress-steps 40 > gpurun_out/r2v/stress4.log 2>&1; echo rc=$? >> gpurun_out/r2v/stress4.log
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2v/ref1.log 2>&1; echo rc=$? >> gpurun_out/r2v/ref1.log
}

recipe_r2w() {
  # multicast / hybrid verification retry: their parity tests, twice
  mkdir -p gpurun_out/r2w
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 400 python -m pytest tests/test_gpu_parity.py -q -rs -k "multicast or hybrid" > gpurun_out/r2w/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2w/pytest_sp.log
  for k in 1 2; do
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -rs -k "17 or 18 or 19 or 21 or 22 or 23" > gpurun_out/r2w/pytest_mp$k.log 2>&1; echo rc=$? >> gpurun_out/r2w/pytest_mp$k.log
  done
}

recipe_r2x() {
  # K-major reshard: double-buffered k_pull_t (12 warps x 2 blocks) vs the round-1 single buffer
  mkdir -p gpurun_out/r2x
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x/build.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "k_major or pull_rules" > gpurun_out/r2x/pytest_kmajor.log 2>&1; echo rc=$? >> gpurun_out/r2x/pytest_kmajor.log
  timeout 300 python tools/pull_bench.py --tps 1,2,4 --layouts k-major > gpurun_out/r2x/pull_dbl.log 2>&1
  LAM_PULL_T_SINGLE=1 timeout 300 python tools/pull_bench.py --tps 1,2,4 --layouts k-major > gpurun_out/r2x/pull_single.log 2>&1
}

recipe_r2y() {
  # HEAD validation on 4 GPUs after the last changes: smoke, pytest -m gpu, bench N=1 and N=4
  mkdir -p gpurun_out/r2y
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2y/smoke.log
  LAM_DEBUG_FAIL=1 timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r2y/pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2y/pytest4.log
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2y/n1.log 2>&1; echo rc=$? >> gpurun_out/r2y/n1.log
  timeout 400 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2y/n4.log 2>&1; echo rc=$? >> gpurun_out/r2y/n4.log
}

recipe_r2z() {
  # two-level broadcast (LAM_HOP_TREE): parity single/multi-process, bench N=2/4 vs the chain
  mkdir -p gpurun_out/r2z
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "tree" > gpurun_out/r2z/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2z/pytest_sp.log
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -rs -k "24 or 25" > gpurun_out/r2z/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2z/pytest_mp.log
  for n in 4 3; do
  timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode tree > gpurun_out/r2z/n${n}_tree.log 2>&1; echo rc=$? >> gpurun_out/r2z/n${n}_tree.log
  done
}

recipe_r2final() {
  # after withdrawing the hybrid mode: smoke, every single-process parity test, the multi-process
  # chain / multicast / tree / host cases
  mkdir -p gpurun_out/r2final
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2final/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2final/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2final/smoke.log
  export LAM_DEBUG_FAIL=1
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream_pull.py -q -rs > gpurun_out/r2final/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2final/pytest_sp.log
  M=tests/test_gpu_multiproc.py::test_multiproc_parity
  timeout 900 python -m pytest -q -rs "$M[0]" "$M[7]" "$M[14]" "$M[17]" "$M[18]" "$M[19]" "$M[21]" "$M[22]" > gpurun_out/r2final/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2final/pytest_mp.log
}

recipe_r2driver() {
  # what the driver runs at round end, on 1 GPU: smoke, pytest -m gpu, bench.py with its K/W
  mkdir -p gpurun_out/r2driver
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2driver/build.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2driver/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2driver/smoke.log
  timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r2driver/pytest1.log 2>&1; echo rc=$? >> gpurun_out/r2driver/pytest1.log
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2driver/n1.log 2>&1; echo rc=$? >> gpurun_out/r2driver/n1.log
}

recipe_r2tree2() {
  # two-level broadcast with the step schedule (node 0 serves one owner per step): parity + bench
  mkdir -p gpurun_out/r2tree2
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2tree2/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "tree" > gpurun_out/r2tree2/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2tree2/pytest_sp.log
  timeout 240 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode tree > gpurun_out/r2tree2/n4_tree.log 2>&1; echo rc=$? >> gpurun_out/r2tree2/n4_tree.log
}

recipe_r2tree3() {
  # two-level broadcast with per-tile flags (a peer's tile is pulled as soon as it landed): parity + bench N=4
  mkdir -p gpurun_out/r2tree3
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2tree3/build.log 2>&1
  export LAM_DEBUG_FAIL=1
  timeout 150 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "tree" > gpurun_out/r2tree3/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/r2tree3/pytest_sp.log
  timeout 150 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --hop-mode tree > gpurun_out/r2tree3/n4_tree.log 2>&1; echo rc=$? >> gpurun_out/r2tree3/n4_tree.log
  M=tests/test_gpu_multiproc.py::test_multiproc_parity
  timeout 200 python -m pytest -q -x -rs "$M[21]" "$M[22]" > gpurun_out/r2tree3/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/r2tree3/pytest_mp.log
}

recipe_r2last() {
  # the chain after the last k_hop change (tile-flag branch): smoke, chain parity across 2 GPUs, bench N=2
  mkdir -p gpurun_out/r2last
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2last/build.log 2>&1
  timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2last/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2last/smoke.log
  timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -rs -k "chain or corrupt or multicast" > gpurun_out/r2last/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2last/pytest.log
  timeout 200 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2last/n2.log 2>&1; echo rc=$? >> gpurun_out/r2last/n2.log
}

recipe_r2fin() {
  # the driver's 1-GPU round-end sequence at HEAD (smoke, pytest -m gpu)
  mkdir -p gpurun_out
  timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2fin_smoke.txt 2>&1
  timeout 220 python -m pytest tests -m gpu -x -q > gpurun_out/r2fin_pytest_gpu.txt 2>&1
}

if [ $# -ne 1 ] || ! declare -F "recipe_$1" > /dev/null; then
  echo "usage: bash tools/gpu_recipes.sh <recipe>; recipes: sweep4 n4 v9 v10 v15 host4 v5 v12 dyn v13 final r2c v14 r2b ncu2 v7 r2d r2a v11 v6 v8 r2e r2f r2g r2h r2j r2l r2m r2n r2o r2p r2q r2r r2s r2t r2u r2v r2w r2x r2y r2z r2final r2driver r2tree2 r2tree3 r2last r2fin"
  exit 2
fi
"recipe_$1"
