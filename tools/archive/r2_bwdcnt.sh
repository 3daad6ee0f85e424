# per-role backward counters (dev counters build), persistent mode
set -u
O=gpurun_out/${1:-r2cnt}; mkdir -p $O
TT_PROFILE_COUNTERS=1 python -m paper_2511_00413_b200.build --dev --force > $O/build_cnt.log 2>&1
timeout 300 python tools/bwdcount.py > $O/bwdcount.txt 2>&1
echo done >> $O/bwdcount.txt
