#!/bin/bash
# FAST 256-wide pair tiles (MTX_TC_BN256=2): parity with the knob, cfg4 N = 1 / 2 / 4 with and without it
mkdir -p gpurun_out/b256
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MTX_TC_BN256=2 CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -q -x -k "3XF16 or f16 or cfg4 or short_input" > gpurun_out/b256/pytest.log 2>&1; tail -2 gpurun_out/b256/pytest.log
for kv in 0 2; do
  MTX_TC_BN256=$kv CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b256/n1_$kv.json 2> gpurun_out/b256/n1_$kv.err
  for n in 2 4; do
    MTX_TC_BN256=$kv timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --config cfg4 --steps 30 --warmup 5 > gpurun_out/b256/n${n}_$kv.json 2> gpurun_out/b256/n${n}_$kv.err
  done
done
python tools/show_bench.py -v gpurun_out/b256/*.json
