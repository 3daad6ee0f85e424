# persistent forward (cluster launch control) A/B: parity, timing with stealing on / off (dev TT_FWD_NOSTEAL),
# sustained clock / power, per-role counters
set -u
O=gpurun_out/${1:-r2g}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attn.py ${PYTEST_EXTRA:-} -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python tools/timeall.py agentic8k wide deep32k > $O/time_release.txt 2>&1
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do
  echo "== steal" >> $O/time.txt; timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
  echo "== nosteal" >> $O/time.txt; TT_FWD_NOSTEAL=1 timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
done
for c in agentic8k deep32k; do
  timeout 120 python tools/attn_power.py $c steal >> $O/power.txt 2>&1
  TT_FWD_NOSTEAL=1 timeout 120 python tools/attn_power.py $c nosteal >> $O/power.txt 2>&1
done
TT_PROFILE_COUNTERS=1 python -m paper_2511_00413_b200.build --dev --force > $O/build_cnt.log 2>&1
echo "== steal" >> $O/fwdcount.txt; timeout 300 python tools/fwdcount.py >> $O/fwdcount.txt 2>&1
echo "== nosteal" >> $O/fwdcount.txt; TT_FWD_NOSTEAL=1 timeout 300 python tools/fwdcount.py >> $O/fwdcount.txt 2>&1
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/time.txt
