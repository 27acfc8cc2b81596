# N=2 cfg2 bench, three back-to-back runs (rank-skew check), and one N=1 run
for i in 1 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$i \
  bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_r$i.json 2> gpurun_out/bench_n2_r$i.err || tail -3 gpurun_out/bench_n2_r$i.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29539 \
  bench.py --gpus 2 --config cfg4 --steps 20 --warmup 5 > gpurun_out/bench_n2_cfg4.json 2> gpurun_out/bench_n2_cfg4.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err || tail -3 gpurun_out/bench_n1.err
