# fwd partial-tile fast path A/B (dev TT_DEBUG_FWD=128 disables it) + attention parity
set -u
O=gpurun_out/${1:-r2fast}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do
  echo "== fast path on" >> $O/time.txt; timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
  echo "== fast path off" >> $O/time.txt; TT_DEBUG_FWD=128 timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/time.txt
