# loss variant A/B inside the bench step (power-capped conditions) + loss parity per variant
set -u
O=gpurun_out/${1:-lossvar}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for v in ${VARS:-1 21 22 23 24}; do
  echo "== TT_LOSS_VARIANT=$v" >> $O/loss.txt
  TT_LOSS_DEBUG=1 TT_LOSS_VARIANT=$v timeout 120 python tools/timeloss.py 2>&1 | sort | uniq | head -4 >> $O/loss.txt
  TT_LOSS_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_loss.py tests/test_gpu_weights.py -x -q -k "loss" 2>&1 | tail -1 >> $O/loss.txt
  for c in agentic8k deep32k; do
    TT_LOSS_VARIANT=$v timeout 300 python bench.py --config $c --steps 5 --no-cpu --no-e2e --no-linear --no-lmhead 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d.get('roofline_loss') or d['roofline']
print('$c', d['value'], d['per_op_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/loss.txt
  done
done
echo done
