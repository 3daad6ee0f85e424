set -u
O=gpurun_out/${1:-r2ad}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do for f in 0 1; do TT_BWD_FLAT=$f timeout 600 python tools/threshold_sweep.py >> $O/sweep.txt 2>&1; done; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/sweep.txt
