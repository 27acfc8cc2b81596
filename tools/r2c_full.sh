#!/bin/bash
# Round-2c full check on a 4-GPU box: smoke, GPU tests (1 GPU), cfg4 N = 1 (x2) / 2 / 4, world-2/4 parity
mkdir -p gpurun_out/full
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full/smoke.log 2>&1; tail -1 gpurun_out/full/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_multigpu.py > gpurun_out/full/pytest_gpu.log 2>&1; tail -2 gpurun_out/full/pytest_gpu.log
for i in 1 2; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/full/n1_$i.json 2> gpurun_out/full/n1_$i.err
done
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/full/n$n.json 2> gpurun_out/full/n$n.err
done
python tools/show_bench.py gpurun_out/full/n*.json
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider > gpurun_out/full/pytest_multigpu.log 2>&1; tail -5 gpurun_out/full/pytest_multigpu.log
