#!/bin/bash
# Round-2b A/B measurements behind DESIGN.md §5 / §13 (one B200 unless noted; outputs in gpurun_out/).
# Usage: bash tools/experiments.sh <name>      e.g. gpurun -- 'bash tools/experiments.sh knobs'
# The prefetch / multicast knobs and MTX_TC_DBG 1-3 exist only in an experiment build, the phase stamps (MTX_TC_DBG=4,
# MTX_FUSED_TS) only in a trace build: this script rebuilds with both (MTX_TC_EXPERIMENTS=1 MTX_TRACE=1); rebuild the
# product library afterwards (build(force=True) without them).
set -x
mkdir -p gpurun_out
MTX_TC_EXPERIMENTS=1 MTX_TRACE=1 python -c "from paper_1704_04560_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
case "$1" in
  knobs)  # GEMM engine knobs on the cfg4 step: L2 prefetch, A multicast, 256-wide pair tiles, CUDA-core first-layer wgrad
    for kv in "" MTX_TC_PF=4 MTX_TC_PF=8 MTX_TC_MC=1 MTX_TC_BN256=1 MTX_SMALLM=1; do
      env $kv timeout 300 python bench.py --no-cpu-baseline > "gpurun_out/knob_${kv:-default}.json" 2>/dev/null
    done
    python tools/show_bench.py -v gpurun_out/knob_*.json ;;
  gemm)   # the cfg4 GEMM shapes alone (3xF16 vs 3xTF32) and with MTX_TC_DBG 1/2/3 (no stores / loads / both)
    for d in 0 1 2 3; do MTX_TC_DBG=$d ENGINE=f16 SHAPES=0,1,2,6,7,8,9,10 python tools/gemm3x_bench.py; done > gpurun_out/exp_gemm.jsonl
    SHAPES=0,1,2 python tools/gemm3x_bench.py >> gpurun_out/exp_gemm.jsonl ;;
  phases) bash tools/tcts.sh ;;  # %globaltimer phase stamps + MMA-warp stall counters (MTX_TC_DBG=4)
  cfg23)  # cfg2 / cfg3 in both split modes (bench --precision auto picks 3xTF32 there)
    for c in cfg2 cfg3; do for p in 3xf16 3xtf32; do
      timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline > gpurun_out/exp_${c}_$p.json 2>/dev/null
    done; done
    python tools/show_bench.py gpurun_out/exp_cfg*.json ;;
  modes4) # 4 GPUs: reduction modes at N = 4 (fused NVLink kernel vs per-bucket NCCL)
    for m in fused nccl; do
      timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 \
        bench.py --gpus 4 --steps 30 --warmup 5 --reduce $m > gpurun_out/exp_mode_$m.json 2>/dev/null
    done
    python tools/show_bench.py gpurun_out/exp_mode_*.json ;;
  fusedts) bash tools/fused_ts.sh ;;  # 4 GPUs: flag wait vs reduction work inside the fused NVLink update
  *) echo "names: knobs gemm phases cfg23 modes4 fusedts" ;;
esac
