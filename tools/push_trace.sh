#!/bin/bash
# simulated-rank tests (fixed build) + fused-kernel wait/work split at P = 2/4 (trace build in tools/alt/trace)
mkdir -p gpurun_out/ptr
timeout 900 python -m pytest tests/test_gpu_simulated_ranks.py tests/test_gpu_determinism.py -q -x > gpurun_out/ptr/pytest_sim.log 2>&1; tail -2 gpurun_out/ptr/pytest_sim.log
cd tools/alt/trace
for n in 2 4; do
  for mode in 1 0; do
    MTX_FUSED_TS=1 MTX_FUSED_PUSH=$mode timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 5 --warmup 3 > ../../../gpurun_out/ptr/n${n}_push$mode.txt 2>&1
  done
done
