#!/bin/bash
# FAST GEMM variants (3xF16, whole-tile fast epilogue only): smoke, GEMM + parity + determinism tests, cfg4 lines
mkdir -p gpurun_out/fc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fc/smoke.log 2>&1; tail -1 gpurun_out/fc/smoke.log
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/fc/pytest.log 2>&1; tail -2 gpurun_out/fc/pytest.log
for i in 1 2; do
  timeout 300 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/fc/cfg4_$i.json 2> gpurun_out/fc/cfg4_$i.err
done
python tools/show_bench.py -v gpurun_out/fc/cfg4_*.json
