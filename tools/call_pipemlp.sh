# loss_pipe_kernel pass-2 loads in flight (TT_PIPE_MLP) A/B, alone and inside the split
set -u
O=gpurun_out/${1:-pipemlp}; mkdir -p $O
for mlp in 4 8 12; do
  TT_EXTRA_NVCC_FLAGS="-DTT_PIPE_MLP=$mlp" python -m paper_2511_00413_b200.build > $O/build_$mlp.log 2>&1
  echo "== TT_PIPE_MLP=$mlp" >> $O/loss.txt
  timeout 300 python -m pytest tests/test_gpu_loss.py -q -k "tail_split or padded or kernel_paths" 2>&1 | tail -1 >> $O/loss.txt
  echo "-- pipe alone" >> $O/loss.txt
  TT_LOSS_VARIANT=0 timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
  for v in 0.7 0.85 1.0; do
    echo "-- split $v" >> $O/loss.txt
    TT_LOSS_SPLIT=$v timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
  done
done
echo done
