#!/bin/bash
# Round-2c final scaling lines on one 4-GPU box: cfg4 N = 1 / 2 / 4 (driver-style launch), cfg2 N = 1 / 2 / 4
mkdir -p gpurun_out/sf
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/sf/topo.txt 2>&1
for cfg in cfg4 cfg2; do
  timeout 400 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sf/${cfg}_n1.json 2> gpurun_out/sf/${cfg}_n1.err
  for n in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config $cfg --steps 30 --warmup 5 > gpurun_out/sf/${cfg}_n$n.json 2> gpurun_out/sf/${cfg}_n$n.err
  done
done
python tools/show_bench.py gpurun_out/sf/*.json
