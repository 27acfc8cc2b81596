# N=2 bench lines (cfg2 default, cfg4) under torchrun
for c in cfg2 cfg4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 2 --config $c --steps 20 --warmup 5 > gpurun_out/bench_n2_$c.json 2> gpurun_out/bench_n2_$c.err || tail -3 gpurun_out/bench_n2_$c.err
done
