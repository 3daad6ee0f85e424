# energy / time share of the backward's per-tile Q / dO loads (flat kernel, dev TT_DEBUG_BWD=2: Q / dO stages
# reused after the first 3 tiles — wrong results, cost measurement only), sustained on batch64k tree 0
set -u
O=gpurun_out/${1:-r2aa}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do
  echo "== normal" >> $O/sustained.txt; TT_SUSTAINED=1 timeout 300 python tools/timeab.py batch64k >> $O/sustained.txt 2>&1
  echo "== no Q/dO reloads" >> $O/sustained.txt; TT_DEBUG_BWD=2 TT_SUSTAINED=1 timeout 300 python tools/timeab.py batch64k >> $O/sustained.txt 2>&1
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/sustained.txt
