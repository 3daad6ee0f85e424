# CTA-order chunk sweep under the power cap (dev build: TT_FWD_CHUNK / TT_BWD_CHUNK), tools/attn_power.py
set -u
O=gpurun_out/${1:-r2chunk}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for c in batch64k deep32k wide agentic8k; do
  for ch in 1 4 16 100000; do
    TT_FWD_CHUNK=$ch TT_BWD_CHUNK=$ch timeout 120 python tools/attn_power.py $c chunk$ch >> $O/power.txt 2>&1
  done
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
