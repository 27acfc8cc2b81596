# N=4 bench lines (cfg2, cfg4) and the N=1/N=2 cfg4 points on the same box
for c in cfg2 cfg4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 4 --config $c --steps 20 --warmup 5 > gpurun_out/bench_n4_$c.json 2> gpurun_out/bench_n4_$c.err || tail -3 gpurun_out/bench_n4_$c.err
done
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1_cfg4.json 2> gpurun_out/bench_n1_cfg4.err
