# round-2 milestone check: build, GPU tests, smoke, default bench line (batch64k), optional extra configs
set -u
O=gpurun_out/${1:-r2}; shift || true
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
for c in "$@"; do timeout 600 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
echo done
