#!/bin/bash
# per-bucket wmax in the overlapped fused reduction: world 2/4 parity, cfg4 N = 4 (and N = 2) lines
mkdir -p gpurun_out/mw
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 4 2; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/mw/n$n.json 2> gpurun_out/mw/n$n.err
done
python tools/show_bench.py -v gpurun_out/mw/n*.json
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider > gpurun_out/mw/pytest_multigpu.log 2>&1; tail -5 gpurun_out/mw/pytest_multigpu.log
