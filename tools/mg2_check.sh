#!/bin/bash
# 2-GPU check: world-2 parity (tests/mp_worker.py: fp32, 3xTF32, 3xF16), smoke, cfg4 bench at N = 1 and 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_mg2.log 2>&1; tail -1 gpurun_out/smoke_mg2.log
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider -k "2" > gpurun_out/pytest_mg2.log 2>&1; tail -2 gpurun_out/pytest_mg2.log
timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/mg_n1_cfg4.json 2> gpurun_out/mg_n1_cfg4.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/mg_n2_cfg4.json 2> gpurun_out/mg_n2_cfg4.err
python tools/show_bench.py -v gpurun_out/mg_n1_cfg4.json gpurun_out/mg_n2_cfg4.json
