#!/bin/bash
# Push-protocol check (gpurun --gpus 4): smoke, simulated-rank reduction tests (pull + push), world 2/4 parity,
# cfg4 N = 1/2/4 with the push protocol (default) and the pull kernel (MTX_FUSED_PUSH=0), same box.
mkdir -p gpurun_out/push
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/push/smoke.log 2>&1; tail -1 gpurun_out/push/smoke.log
timeout 900 python -m pytest tests/test_gpu_simulated_ranks.py tests/test_gpu_determinism.py -q -x > gpurun_out/push/pytest_sim.log 2>&1; tail -2 gpurun_out/push/pytest_sim.log
timeout 400 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/push/n1.json 2> gpurun_out/push/n1.err
for n in 2 4; do
  for mode in 1 0; do
    MTX_FUSED_PUSH=$mode timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/push/n${n}_push$mode.json 2> gpurun_out/push/n${n}_push$mode.err
  done
done
for f in gpurun_out/push/*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
    print('$f', d['ms_per_step'], d['value'], d.get('replicas_bit_identical'), {k:v for k,v in r['launches_us_per_step'].items() if 'fused' in k or 'barrier' in k or 'push' in k})
except Exception as e: print('$f', 'ERR', e)"; done
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider > gpurun_out/push/pytest_multigpu.log 2>&1; tail -4 gpurun_out/push/pytest_multigpu.log
