# loss head/tail split A/B (TT_LOSS_SPLIT = pipe/cluster per-SM row-rate ratio; 0 = clusters only)
set -u
O=gpurun_out/${1:-split}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loss.py tests/test_gpu_weights.py tests/test_gpu_random_sweep.py -q -k "loss" > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
echo "== TT_LOSS_VARIANT=0 (loss_pipe_kernel alone, all rows)" >> $O/loss.txt
TT_LOSS_VARIANT=0 timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
for v in ${VALS:-0 0.5 0.75 1.0 1.25}; do
  echo "== TT_LOSS_SPLIT=$v" >> $O/loss.txt
  TT_LOSS_SPLIT=$v timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
  TT_LOSS_SPLIT=$v timeout 300 python bench.py --steps 5 --no-cpu --no-e2e --no-linear --no-lmhead 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('agentic8k', d['value'], d['per_op_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/loss.txt
done
echo done
