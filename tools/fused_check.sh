#!/bin/bash
# fused reduction kernel change: simulated-rank + determinism tests, cfg4 N = 4 / 2 lines, world-2/4 parity
mkdir -p gpurun_out/fk
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fk/smoke.log 2>&1; tail -1 gpurun_out/fk/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_simulated_ranks.py tests/test_gpu_determinism.py -q -x > gpurun_out/fk/pytest_sim.log 2>&1; tail -2 gpurun_out/fk/pytest_sim.log
for n in 4 2; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/fk/n$n.json 2> gpurun_out/fk/n$n.err
done
python tools/show_bench.py gpurun_out/fk/n*.json
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider > gpurun_out/fk/pytest_multigpu.log 2>&1; tail -5 gpurun_out/fk/pytest_multigpu.log
