#!/bin/bash
# Multi-GPU run (gpurun --gpus 4): multi-GPU parity tests, cfg5 sweep at P=2/4, bench scaling N=1/2/4.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q > gpurun_out/pytest_mgpu.log 2>&1; tail -3 gpurun_out/pytest_mgpu.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N tools/cfg5_sweep.py > gpurun_out/cfg5_P$N.log 2>&1; tail -12 gpurun_out/cfg5_P$N.log
done
for cfg in cfg2 cfg3 cfg4; do
  for N in 1 2 4; do
    if [ $N = 1 ]; then
      timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/scale_${cfg}_N$N.json 2> gpurun_out/scale_${cfg}_N$N.err
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --config $cfg --gpus $N --steps 30 --warmup 5 > gpurun_out/scale_${cfg}_N$N.json 2> gpurun_out/scale_${cfg}_N$N.err
    fi
    python -c "import json; d=json.load(open('gpurun_out/scale_${cfg}_N$N.json')); print('$cfg', $N, d['value'], d['ms_per_step'], d['per_rank_ms'], d['e2e']['value'])" || tail -3 gpurun_out/scale_${cfg}_N$N.err
  done
done
