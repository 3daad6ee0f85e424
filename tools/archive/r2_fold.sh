# tree-scale fold A/B (dev TT_BWD_NOFOLD) under the power cap + full GPU suite incl. the 2-rank bench test
set -u
O=gpurun_out/${1:-r2fold}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do for c in deep32k batch64k; do
  timeout 120 python tools/attn_power.py $c fold >> $O/power.txt 2>&1
  TT_BWD_NOFOLD=1 timeout 120 python tools/attn_power.py $c nofold >> $O/power.txt 2>&1
done; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
