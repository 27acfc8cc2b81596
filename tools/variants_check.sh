#!/bin/bash
# epilogue-mode GEMM variants: smoke, GEMM/parity/determinism tests, cfg4 / cfg2 / cfg3 lines
mkdir -p gpurun_out/vc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/vc/smoke.log 2>&1; tail -1 gpurun_out/vc/smoke.log
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/vc/pytest.log 2>&1; tail -2 gpurun_out/vc/pytest.log
for c in cfg4 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/vc/$c.json 2> gpurun_out/vc/$c.err
done
python tools/show_bench.py -v gpurun_out/vc/*.json
