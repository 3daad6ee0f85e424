# idle-warp wait A/B on the attention kernels (dev build): batch64k tree 0 back to back (power-capped)
set -u
O=gpurun_out/${1:-r2waitattn}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for rep in 1 2; do for w in 0 2 3 7; do echo "== TT_WAIT_HINT=$w" >> $O/time.txt; TT_WAIT_HINT=$w timeout 300 python tools/timeall.py batch64k >> $O/time.txt 2>&1; done; done
python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
echo done
