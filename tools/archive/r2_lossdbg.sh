set -u
O=gpurun_out/${1:-r2lossdbg}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for v in 25 21; do echo "== $v" >> $O/dbg.txt; TT_LOSS_VARIANT=$v timeout 120 python tools/loss_fp16_debug.py >> $O/dbg.txt 2>&1; done
echo done
