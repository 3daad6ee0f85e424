# forward polynomial-exponential share at the power cap (compile-time TT_FWD_POLY 0 / 1 (shipped) / 2), batch64k tree 0
set -u
O=gpurun_out/${1:-r2ac}; mkdir -p $O
for pp in 1 0 2 1; do
  TT_EXTRA_NVCC_FLAGS="-DTT_FWD_POLY=$pp" python -m paper_2511_00413_b200.build --dev --force > $O/build_$pp.log 2>&1
  echo "== TT_FWD_POLY=$pp" >> $O/sustained.txt; TT_SUSTAINED=1 timeout 300 python tools/timeab.py batch64k >> $O/sustained.txt 2>&1
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/sustained.txt
