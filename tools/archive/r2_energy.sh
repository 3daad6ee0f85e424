# energy-per-FLOP A/B under the power cap (sustained kernels, tools/attn_power.py), dev builds
set -u
O=gpurun_out/${1:-r2en}; mkdir -p $O
run() { for c in deep32k batch64k; do timeout 120 python tools/attn_power.py $c "$1" >> $O/power.txt 2>&1; done; }
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
run base
TT_CTA_ORDER=2 timeout 120 python tools/attn_power.py batch64k bwd-head-major >> $O/power.txt 2>&1
TT_EXTRA_NVCC_FLAGS="-DTT_BWD_POLY=0 -DTT_FWD_POLY=0" python -m paper_2511_00413_b200.build --dev --force >> $O/build.log 2>&1
run poly0
TT_EXTRA_NVCC_FLAGS="-DTT_BWD_POLY=2 -DTT_FWD_POLY=2" python -m paper_2511_00413_b200.build --dev --force >> $O/build.log 2>&1
run poly2
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
