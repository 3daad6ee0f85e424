set -u
O=gpurun_out/${1:-losssm}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for c in 33 28 24 20 16; do echo "== clusters $c" >> $O/loss.txt; TT_LOSS_MAXCL=$c timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1; TT_LOSS_NOCOMPUTE=1 TT_LOSS_MAXCL=$c timeout 120 python tools/timeloss.py 2>&1 | sed 's/^/nocompute /' >> $O/loss.txt; done
echo done
