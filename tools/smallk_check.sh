#!/bin/bash
# fwd_smallk change: parity tests that reach it (3xF16 small-K first layers) + cfg4 N=1 lines
mkdir -p gpurun_out/sk
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/sk/pytest.log 2>&1; tail -2 gpurun_out/sk/pytest.log
for i in 1 2; do
  timeout 300 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sk/cfg4_$i.json 2> gpurun_out/sk/cfg4_$i.err
done
python tools/show_bench.py -v gpurun_out/sk/cfg4_*.json
