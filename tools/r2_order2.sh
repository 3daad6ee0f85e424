# CTA order with the persistent kernels on agentic8k / wide: heuristic vs forced head-major (dev TT_CTA_ORDER=3)
set -u
O=gpurun_out/${1:-r2y}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do
  echo "== heuristic" >> $O/time.txt; timeout 300 python tools/timeab.py agentic8k wide >> $O/time.txt 2>&1
  echo "== head-major" >> $O/time.txt; TT_CTA_ORDER=3 timeout 300 python tools/timeab.py agentic8k wide >> $O/time.txt 2>&1
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/time.txt
