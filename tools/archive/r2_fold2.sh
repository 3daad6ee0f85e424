# full GPU suite after the fold-for-non-negative-weights change + per-role cycle counters (dev build)
set -u
O=gpurun_out/${1:-r2fold2}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
TT_PROFILE_COUNTERS=1 python -m paper_2511_00413_b200.build --dev --force > $O/build_cnt.log 2>&1
timeout 300 python tools/bwdcount.py > $O/bwdcount.txt 2>&1
timeout 300 python tools/fwdcount.py > $O/fwdcount.txt 2>&1
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/fwdcount.txt
