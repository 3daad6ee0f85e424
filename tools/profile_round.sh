#!/bin/bash
# One GPU call: tests, bench lines per config, launch list and ncu --set full of the top kernels.
#   gpurun --timeout 2400 -- 'bash tools/profile_round.sh r1'
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_agentic8k.json 2> $O/bench_agentic8k.err
for c in deep32k wide batch64k; do
  timeout 600 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_agentic8k.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-linear --no-lmhead > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' \
  --launch-skip 12 --launch-count 4 -o $O/full_agentic8k -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-linear --no-lmhead > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100' \
  --launch-skip 6 --launch-count 2 -o $O/full_deep32k -f \
  python bench.py --config deep32k --steps 1 --warmup 3 --no-cpu --no-e2e --no-linear --no-lmhead --no-loss > $O/ncu_full32.log 2>&1
echo done
