# round-2 profile call: GPU tests, smoke, driver-style bench line (batch64k), launch list, ncu --set full
#   gpurun --timeout 3600 -- 'bash tools/r2_prof.sh r2c'
set -u
TAG=${1:-r2c}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
timeout 600 python bench.py --config agentic8k --steps 20 --warmup 5 --no-cpu > $O/bench_agentic8k.json 2> $O/bench_agentic8k.err
# launch list of one batch64k step on 4 trees (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_batch64k.csv \
  python bench.py --trees 4 --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
# ncu --set full of tree 0's fwd / loss / bwd (after 3 warm-up steps)
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' --launch-skip 12 --launch-count 4 \
  -o $O/full_batch64k -f python bench.py --trees 1 --steps 1 --warmup 3 --no-extras > $O/ncu_full.log 2>&1
# ncu --set full of the LM-head GEMMs (sweep 1 over the vocabulary + one chunk's three)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_pair_kernel' --launch-skip 4 --launch-count 4 \
  -o $O/full_gemm -f python tools/timegemm.py --lmhead-only > $O/ncu_gemm.log 2>&1
echo done
