#!/bin/bash
# cfg4 bench lines at N = 1, 2, 4 on one 4-GPU box (3xF16 default), fused NVLink reduction at N > 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/s_n1.json 2> gpurun_out/s_n1.err
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --steps 30 --warmup 5 > gpurun_out/s_n$n.json 2> gpurun_out/s_n$n.err
done
python tools/show_bench.py -v gpurun_out/s_n1.json gpurun_out/s_n2.json gpurun_out/s_n4.json
