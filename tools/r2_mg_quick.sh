#!/bin/bash
# Quick multi-GPU iteration: world-N parity test (optional) + cfg4 / cfg2 bench lines at N GPUs for a few
# MTX_COMM_SMS settings.  Usage: tools/r2_mg_quick.sh N [test] [sms...]
N=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
if [ "$1" = "test" ]; then
  shift
  timeout 900 python -m pytest tests/test_multigpu.py -m gpu -v -p no:cacheprovider -k "[$N]" > gpurun_out/pytest_mg_quick_$N.log 2>&1
  tail -3 gpurun_out/pytest_mg_quick_$N.log
fi
for sms in "${@:-16}"; do
  for cfg in cfg4 cfg2; do
    MTX_COMM_SMS=$sms timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus $N --config $cfg --steps 30 --warmup 5 > gpurun_out/q_n${N}_${cfg}_s$sms.json 2> gpurun_out/q_n${N}_${cfg}_s$sms.err
    python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/q_n${N}_${cfg}_s$sms.json').read().strip().splitlines()[-1])
    r=d['roofline']['breakdown_us_per_step']
    print('N=$N $cfg sms=$sms', d['ms_per_step'], d['per_rank_ms'], d['replicas_bit_identical'], {k: r[k] for k in list(r)[:6]})
except Exception as e: print('N=$N $cfg sms=$sms FAILED', e); print(open('gpurun_out/q_n${N}_${cfg}_s$sms.err').read()[-1500:])
"
  done
done
