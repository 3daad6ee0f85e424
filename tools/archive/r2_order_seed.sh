set -u
O=gpurun_out/${1:-r2os}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for s in 0 2 3; do for ch in 1 100000; do
  TT_FWD_CHUNK=$ch TT_BWD_CHUNK=$ch timeout 120 python tools/order_seed.py deep32k $s chunk$ch >> $O/power.txt 2>&1
done; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
