# 2-GPU check: build, multi-GPU parity tests, bench N=2 (torchrun, NCCL)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 900 python -m pytest tests -m multigpu -q -x > gpurun_out/pytest_multigpu.log 2>&1; tail -3 gpurun_out/pytest_multigpu.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; tail -2 gpurun_out/bench_n2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --config cfg4 --steps 20 --warmup 5 > gpurun_out/bench_n2_cfg4.json 2> gpurun_out/bench_n2_cfg4.err; tail -2 gpurun_out/bench_n2_cfg4.err
