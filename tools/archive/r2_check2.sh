# full GPU suite + sustained attention (release, CTA-order heuristic) + dQ-reduce energy ablations (dev)
set -u
O=gpurun_out/${1:-r2c2}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in batch64k deep32k wide agentic8k; do timeout 120 python tools/attn_power.py $c release >> $O/power.txt 2>&1; done
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for dbg in 32 1; do TT_DEBUG_BWD=$dbg timeout 120 python tools/attn_power.py deep32k dbg$dbg >> $O/power.txt 2>&1; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
