# loss: parity (loss + random sweep) and timing, shipped variant vs round 1's (dev build A/B)
set -u
O=gpurun_out/${1:-r2loss}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loss.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py tests/test_gpu_pack.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
echo "== release (variant 25)" > $O/time.txt
timeout 300 python tools/timeloss.py agentic8k wide deep32k >> $O/time.txt 2>&1
python -m paper_2511_00413_b200.build --dev --force >> $O/build.log 2>&1
for v in 21 25; do echo "== dev TT_LOSS_VARIANT=$v" >> $O/time.txt; TT_LOSS_VARIANT=$v timeout 300 python tools/timeloss.py agentic8k wide deep32k >> $O/time.txt 2>&1; done
python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
echo done
