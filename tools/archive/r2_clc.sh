# cluster-launch-control order probe; same-box A/B of the round-2 start kernels (ab_old = git archive c93e53d)
# against the persistent ones, short bursts and sustained (power-capped)
set -u
O=gpurun_out/${1:-r2o}; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o $O/clc_probe tools/clc_probe.cu > $O/probe_build.log 2>&1
timeout 120 $O/clc_probe > $O/clc_probe.txt 2>&1
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
(cd ab_old && python -m paper_2511_00413_b200.build --force > ../$O/build_old.log 2>&1)
for r in 1 2; do
  TT_ROOT=/root/repo timeout 300 python tools/timeab.py batch64k deep32k:0 deep32k:1 agentic8k wide >> $O/time.txt 2>&1
  TT_ROOT=/root/repo/ab_old timeout 300 python tools/timeab.py batch64k deep32k:0 deep32k:1 agentic8k wide >> $O/time.txt 2>&1
done
TT_SUSTAINED=1 TT_ROOT=/root/repo timeout 300 python tools/timeab.py batch64k deep32k:0 > $O/sustained.txt 2>&1
TT_SUSTAINED=1 TT_ROOT=/root/repo/ab_old timeout 300 python tools/timeab.py batch64k deep32k:0 >> $O/sustained.txt 2>&1
echo done >> $O/time.txt
