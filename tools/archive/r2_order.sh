# bwd issue-order A/B (dev TT_BWD_ORDER=1: dP(i+1) before dK(i)) under the power cap + parity with it
set -u
O=gpurun_out/${1:-r2ord}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
TT_BWD_ORDER=1 timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for r in 1 2; do for c in deep32k batch64k agentic8k; do
  timeout 120 python tools/attn_power.py $c order0 >> $O/power.txt 2>&1
  TT_BWD_ORDER=1 timeout 120 python tools/attn_power.py $c order1 >> $O/power.txt 2>&1
done; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
