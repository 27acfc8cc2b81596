#!/bin/bash
# cfg4 N = 4: per-bucket overlapped fused reduction with MTX_COMM_SMS reserved SMs vs one launch after the backward
mkdir -p gpurun_out/ovs
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  for kv in "MTX_FUSED_OVERLAP=0" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=4" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=8" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=12" "MTX_FUSED_OVERLAP=1 MTX_COMM_SMS=16"; do
    tag=$(echo "$kv" | tr ' =' '__')_$rep
    env $kv timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus 4 --config cfg4 --steps 30 --warmup 5 > gpurun_out/ovs/$tag.json 2> gpurun_out/ovs/$tag.err
  done
done
for f in gpurun_out/ovs/*.json; do python -c "
import json
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3,1), d['value'], d.get('replicas_bit_identical'))
except Exception as e: print('$f ERR', e)"; done
