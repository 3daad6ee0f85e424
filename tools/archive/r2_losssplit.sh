# loss head/tail split ratio sweep (dev TT_LOSS_SPLIT) on agentic8k / wide / deep32k at V = 151,936
set -u
O=gpurun_out/${1:-r2ls}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for r in 1 2; do for sp in 0.6 0.65 0.7 0.75 0.8 0.9; do
  echo "== split $sp" >> $O/split.txt; TT_LOSS_SPLIT=$sp timeout 300 python tools/timeloss.py agentic8k wide deep32k >> $O/split.txt 2>&1
done; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/split.txt
