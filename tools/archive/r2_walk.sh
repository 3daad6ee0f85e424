# bwd query-walk A/B (dev build): time + DRAM bytes per launch
set -u
O=gpurun_out/${1:-r2walk}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for w in 0 1 2 3; do echo "== TT_BWD_WALK=$w" >> $O/time.txt; TT_BWD_WALK=$w timeout 300 python tools/timeall.py batch64k deep32k agentic8k >> $O/time.txt 2>&1; done
for w in 0 1 3; do
  TT_BWD_WALK=$w timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:tree_attn_bwd_sm100 --launch-skip 3 --launch-count 1 --csv python tools/timeall.py batch64k > $O/ncu_walk$w.csv 2>&1
done
python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
echo done
