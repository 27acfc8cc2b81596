#!/bin/bash
# overlap default check: cfg2 and cfg4 at N = 4, MTX_FUSED_OVERLAP = 0 / 1, alternating, two repeats
mkdir -p gpurun_out/oc
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do for cfg in cfg2 cfg4; do for ov in 0 1; do
  MTX_FUSED_OVERLAP=$ov timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus 4 --config $cfg --steps 30 --warmup 5 > gpurun_out/oc/${cfg}_ov${ov}_$rep.json 2> gpurun_out/oc/${cfg}_ov${ov}_$rep.err
done; done; done
python tools/show_bench.py gpurun_out/oc/*.json
