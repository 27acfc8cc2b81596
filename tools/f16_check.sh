#!/bin/bash
# 3xF16 bring-up on one B200: kernel-level parity, step parity, then the cfg4 bench in both split modes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f16_build.log 2>&1 || { tail -20 gpurun_out/f16_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "3xf16" -p no:cacheprovider > gpurun_out/f16_gemm.log 2>&1; tail -3 gpurun_out/f16_gemm.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -p no:cacheprovider > gpurun_out/f16_parity.log 2>&1; tail -15 gpurun_out/f16_parity.log
timeout 300 python bench.py --precision 3xf16 --no-cpu-baseline > gpurun_out/f16_bench_cfg4.json 2> gpurun_out/f16_bench_cfg4.err; tail -3 gpurun_out/f16_bench_cfg4.err
timeout 300 python bench.py --precision 3xf16 --no-cpu-baseline --config cfg2 > gpurun_out/f16_bench_cfg2.json 2> gpurun_out/f16_bench_cfg2.err; tail -3 gpurun_out/f16_bench_cfg2.err
python tools/show_bench.py -v gpurun_out/f16_bench_cfg4.json gpurun_out/f16_bench_cfg2.json
