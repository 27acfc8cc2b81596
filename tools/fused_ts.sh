#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 2 4; do
  MTX_FUSED_TS=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/fts_n$n.json 2> gpurun_out/fts_n$n.err
  grep -h fusedts gpurun_out/fts_n$n.json gpurun_out/fts_n$n.err | tail -24 > gpurun_out/fts_n$n.txt
done
