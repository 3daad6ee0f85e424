# forward 64-key sub-steps with double-buffered S (dev TT_FWD_SUB64=1) vs the shipped 128-key form
set -u
O=gpurun_out/${1:-r2sub}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
TT_FWD_SUB64=1 timeout 600 python tools/timeall.py agentic8k > $O/smoke_time.txt 2>&1; echo "exit $?" >> $O/smoke_time.txt
TT_FWD_SUB64=1 timeout 1500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py tests/test_gpu_block.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for r in 1 2; do
  echo "== sub64" >> $O/time.txt; TT_FWD_SUB64=1 timeout 300 python tools/timeall.py agentic8k wide deep32k batch64k >> $O/time.txt 2>&1
  echo "== 128" >> $O/time.txt; TT_FWD_SUB64=0 timeout 300 python tools/timeall.py agentic8k wide deep32k batch64k >> $O/time.txt 2>&1
done
for c in deep32k batch64k agentic8k; do
  TT_FWD_SUB64=1 timeout 120 python tools/attn_power.py $c sub64 >> $O/power.txt 2>&1
  TT_FWD_SUB64=0 timeout 120 python tools/attn_power.py $c k128 >> $O/power.txt 2>&1
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
