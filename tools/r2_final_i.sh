# final verification of the shipped build (full GPU suite, smoke, default + agentic8k bench lines) and a
# claim / prepare look-ahead sweep of the persistent kernels on agentic8k (dev builds, compile-time)
set -u
O=gpurun_out/${1:-r2w}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
timeout 600 python bench.py --config agentic8k --steps 20 --warmup 5 --no-cpu > $O/bench_agentic8k.json 2> $O/bench_agentic8k.err
for cfg in "5 3 6 3" "3 2 4 2" "8 4 10 4" "2 1 3 1"; do
  set -- $cfg
  TT_EXTRA_NVCC_FLAGS="-DTT_FWD_CLAIM_AHEAD=$1 -DTT_FWD_PREPARE_AHEAD=$2 -DTT_BWD_CLAIM_AHEAD=$3 -DTT_BWD_PREPARE_AHEAD=$4" \
    python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
  for r in 1 2; do echo "== fwd claim/prepare $1/$2 bwd $3/$4" >> $O/ahead.txt; timeout 300 python tools/timeab.py agentic8k wide >> $O/ahead.txt 2>&1; done
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done > $O/done.txt
