set -u
O=gpurun_out/${1:-smoke}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=compute_mode,persistence_mode --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
for i in 1 2 3; do timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt; done
echo done
