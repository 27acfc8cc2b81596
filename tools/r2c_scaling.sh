#!/bin/bash
# Round-2c scaling check (gpurun --gpus 4): cfg4 N = 1/2/4 (default precision, fused pull reduction), cfg2 N = 1
# in both fp32-tier tensor-core modes, cfg3 N = 1 in both, world-2/4 parity (pull + push).
mkdir -p gpurun_out/sc
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 400 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sc/cfg4_n1.json 2> gpurun_out/sc/cfg4_n1.err
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/sc/cfg4_n$n.json 2> gpurun_out/sc/cfg4_n$n.err
done
for c in cfg2 cfg3; do for p in 3xtf32 3xf16; do
  timeout 400 python bench.py --config $c --precision $p --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sc/${c}_$p.json 2> gpurun_out/sc/${c}_$p.err
done; done
for f in gpurun_out/sc/*.json; do python -c "
import json
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step']*1e3,1), d['value'], d.get('replicas_bit_identical'), d['clocks'])
except Exception as e: print('$f ERR', e)"; done
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider > gpurun_out/sc/pytest_multigpu.log 2>&1; tail -5 gpurun_out/sc/pytest_multigpu.log
