set -u
O=gpurun_out/${1:-lossnc}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
echo "== normal" > $O/loss.txt; timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
echo "== no compute (pure TMA stream through smem)" >> $O/loss.txt; TT_LOSS_NOCOMPUTE=1 timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
python - >> $O/loss.txt 2>&1 <<'PY'
import torch
x = torch.empty(8192 * 151936, dtype=torch.bfloat16, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
for _ in range(10): y.copy_(x)
b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b) / 10
print(f"torch copy of the agentic8k logits: {ms:.3f} ms  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
PY
echo done
