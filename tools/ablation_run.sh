#!/bin/bash
# 4-GPU call: multi-GPU tests, then the reduce-mode ablation (bench lines per mode, N = 2, 4)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q > gpurun_out/pytest_mgpu.log 2>&1; tail -2 gpurun_out/pytest_mgpu.log
grep -o '"error": "[^"]*' gpurun_out/pytest_mgpu.log | head -3
for c in ${CONFIGS:-cfg2 cfg4}; do for N in 2 4; do for r in ${MODES:-nccl fused layerwise zero1}; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --config $c --gpus $N --steps 30 --warmup 5 --reduce $r > gpurun_out/abl_${c}_n${N}_$r.json 2> gpurun_out/abl_${c}_n${N}_$r.err
  echo -n "$c N=$N $r: "; python tools/show_bench.py gpurun_out/abl_${c}_n${N}_$r.json | head -1 | cut -c1-150
done; done; done
