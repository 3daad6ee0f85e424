set -u
O=gpurun_out/${1:-bwdcount}; mkdir -p $O
TT_PROFILE_COUNTERS=1 python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 300 python tools/bwdcount.py > $O/counters.txt 2>&1
echo done
