set -u
O=gpurun_out/${1:-alt}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py -x -q -k "bf16 or tensor_core or full_size or edge" > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
echo "== ALTERNATE=1" > $O/time.txt; timeout 200 python tools/timefwd.py >> $O/time.txt 2>&1
TT_EXTRA_NVCC_FLAGS="-DTT_FWD_ALTERNATE=0" python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
echo "== ALTERNATE=0" >> $O/time.txt; timeout 200 python tools/timefwd.py >> $O/time.txt 2>&1
echo done
