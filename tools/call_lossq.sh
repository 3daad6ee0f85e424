set -u
O=gpurun_out/${1:-lossq}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for v in ${VARS}; do echo "== $v" >> $O/loss.txt; TT_LOSS_DEBUG=1 TT_LOSS_VARIANT=$v timeout 120 python tools/timeloss.py 2>&1 | sort | uniq | head -4 >> $O/loss.txt; done
echo done
