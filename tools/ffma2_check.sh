#!/bin/bash
# FFMA2 (packed fp32 FMA) in fwd_smallk and conv_wgrad: parity + cfg4 / cfg3 lines
mkdir -p gpurun_out/f2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f2/smoke.log 2>&1; tail -1 gpurun_out/f2/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/f2/pytest.log 2>&1; tail -2 gpurun_out/f2/pytest.log
for i in 1 2; do
  timeout 300 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/f2/cfg4_$i.json 2> gpurun_out/f2/cfg4_$i.err
  timeout 300 python bench.py --config cfg3 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/f2/cfg3_$i.json 2> gpurun_out/f2/cfg3_$i.err
done
python tools/show_bench.py -v gpurun_out/f2/cfg4_*.json gpurun_out/f2/cfg3_*.json
