#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider -k "2" > gpurun_out/pytest_mg2.log 2>&1; tail -3 gpurun_out/pytest_mg2.log
