# round-2 (second session) profile call: smoke, driver-style bench lines, launch list, ncu --set full
#   gpurun --timeout 3600 -- 'bash tools/r2_prof2.sh r2e'
set -u
TAG=${1:-r2e}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
for c in agentic8k deep32k wide; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_batch64k.csv \
  python bench.py --trees 4 --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' --launch-skip 12 --launch-count 4 \
  -o $O/full_batch64k -f python bench.py --trees 1 --steps 1 --warmup 3 --no-extras > $O/ncu_full.log 2>&1
echo done > $O/done.txt
