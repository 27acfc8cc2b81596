#!/bin/bash
# Round-2 multi-GPU check (gpurun --gpus 4): the world-2/4 parity tests (tests/mp_worker.py), then cfg4 and
# cfg2 bench lines at N = 2 and 4 (torchrun, fused NVLink reduction) and the N = 1 line on the same box.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider > gpurun_out/pytest_multigpu_r2.log 2>&1; tail -4 gpurun_out/pytest_multigpu_r2.log
for cfg in cfg4 cfg2; do
  timeout 400 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/mg_n1_$cfg.json 2> gpurun_out/mg_n1_$cfg.err
  for n in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config $cfg --steps 30 --warmup 5 > gpurun_out/mg_n${n}_$cfg.json 2> gpurun_out/mg_n${n}_$cfg.err
  done
done
ls -la gpurun_out/mg_*
