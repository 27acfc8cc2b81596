#!/bin/bash
# cfg4 N = 2/4: one fused launch after the backward (default) vs the per-bucket overlapped ablation
# (MTX_FUSED_OVERLAP=1, MTX_COMM_SMS SMs reserved), same box
mkdir -p gpurun_out/ov
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 4 2; do
  for kv in "MTX_FUSED_OVERLAP=0" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=20" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=12" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=32"; do
    tag=$(echo "$kv" | tr ' =' '__')
    env $kv timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/ov/n${n}_$tag.json 2> gpurun_out/ov/n${n}_$tag.err
  done
done
for f in gpurun_out/ov/*.json; do python -c "
import json
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3,1), d['value'], d.get('replicas_bit_identical'))
except Exception as e: print('$f ERR', e)"; done
