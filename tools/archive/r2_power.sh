# power / clock of the sustained attention kernels, release build and backward ablations (dev build)
set -u
O=gpurun_out/${1:-r2pow}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
for c in deep32k batch64k agentic8k; do timeout 120 python tools/attn_power.py $c release >> $O/power.txt 2>&1; done
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for dbg in 1 4 5; do TT_DEBUG_BWD=$dbg timeout 120 python tools/attn_power.py deep32k dbg$dbg >> $O/power.txt 2>&1; done
TT_EXTRA_NVCC_FLAGS="-DTT_BWD_VTMEM=0" python -m paper_2511_00413_b200.build --dev --force > $O/build0.log 2>&1
timeout 120 python tools/attn_power.py deep32k vtmem0 >> $O/power.txt 2>&1
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
