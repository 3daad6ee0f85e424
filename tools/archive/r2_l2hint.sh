# L2 eviction-policy A/B of the backward (dev build TT_BWD_L2HINT) under the power cap + ncu DRAM bytes
set -u
O=gpurun_out/${1:-r2l2}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for hnt in 0 1 2 4 5 0; do for c in deep32k batch64k; do
  TT_BWD_L2HINT=$hnt timeout 120 python tools/attn_power.py $c hint$hnt >> $O/power.txt 2>&1; done; done
for hnt in 0 1 5; do
  TT_BWD_L2HINT=$hnt timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:tree_attn_bwd -c 1 --csv python tools/one_bwd.py deep32k > $O/ncu_hint$hnt.csv 2>&1
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
